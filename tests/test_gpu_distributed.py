"""Multi-rank path end to end on the GPU: two processes (gloo, both on GPU 0 --
the rank logic is the same as one GPU per rank with NCCL) each contract their
contiguous slice block with the B200 executor through
``contract_sliced_distributed``; the all-reduced sum must equal the oracle's
full sliced sum on every rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    from paper_2002_01935_b200.harness import generators as gen
    from paper_2002_01935_b200.harness.paths import best_greedy_tree
    from paper_2002_01935_b200.slicing import greedy_slice
    from paper_2002_01935_b200.refpkg import metrics
    tn = gen.random_regular(30, 3, seed=9)
    # two open legs, so the all-reduce carries a tensor, not a scalar
    tn = tn.replace(output=tuple(list(tn.index_table)[:2]))
    tree = best_greedy_tree(tn, trials=2)
    ss = greedy_slice(tree, tn, metrics(tree, tn).width - 3, restarts=1)
    return tn, tree, ss


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2002_01935_b200.distributed import contract_sliced_distributed
        tn, tree, ss = _case()
        total = contract_sliced_distributed(tn, tree, ss)
        q.put((rank, np.asarray(total, dtype=np.complex128).tolist() if np.ndim(total) else complex(total)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_contract_sliced_distributed_gloo_ranks_share_gpu(world):
    import oracle
    tn, tree, ss = _case()
    assert ss.d >= world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = sorted((q.get() for _ in range(world)), key=lambda t: t[0])
    ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels)
    ref = np.asarray(ref, dtype=np.complex128)
    vals = [np.asarray(v, dtype=np.complex128) for _, v in res]
    for v in vals:
        assert np.linalg.norm((v - ref).ravel()) <= 1e-5 * max(np.linalg.norm(ref.ravel()), 1e-30)
    for v in vals[1:]:
        assert np.array_equal(v, vals[0])
