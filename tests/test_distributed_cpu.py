"""World-size-2 gloo tests of the multi-rank path on CPU: contiguous slice
partition, per-rank partial sums (oracle stand-in for the device partials)
and the single complex128 all-reduce reproduce the full sliced sum."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2002_01935_b200.distributed import slice_range


def test_slice_range_partition():
    for d in (1, 2, 7, 16, 1000):
        for world in (1, 2, 3, 4, 8):
            blocks = [slice_range(0, d, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == d
            for (a, b), (c, e) in zip(blocks, blocks[1:]):
                assert b == c
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    big = 1 << 60
    lo, hi = slice_range(0, big, 8, 7)
    assert hi == big and lo == 7 * (big // 8)
    with pytest.raises(ValueError):
        slice_range(0, 4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2002_01935_b200.distributed import allreduce_complex, slice_range
        from paper_2002_01935_b200.harness import generators as gen
        from paper_2002_01935_b200.harness.paths import greedy_tree
        tn = gen.random_hyper_network(7, 12, seed=11, p_output=0.5)
        tree = greedy_tree(tn)
        S = [l for l in tn.index_table if l not in tn.output][:3]
        d = int(np.prod([tn.index_table[l] for l in S]))
        lo, hi = slice_range(0, d, world, rank)
        part, _, _ = oracle.contract_sliced(tn, tree, S, slice_ids=range(lo, hi)) if hi > lo else (0.0, 0, 0)
        if hi == lo:
            full_shape = np.shape(oracle.contract(tn, tree)[0])
            part = np.zeros(full_shape, dtype=np.complex128)
        total = allreduce_complex(part)
        ref, _, _ = oracle.contract_sliced(tn, tree, S)
        q.put((rank, float(np.max(np.abs(np.asarray(total) - np.asarray(ref))))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_allreduce_of_partials(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    for rank, err in res:
        assert err <= 1e-12, (rank, err)
