"""Randomised parity sweep (GPU vs the complex128 oracle) over networks big
enough to reach the tensor-core paths: 3/4-regular graphs, small grid
circuits (split and diagonal-reduced) and hypergraph networks with open outputs, random greedy trees,
random slicings, random precision / fusion options, lowered GEMM thresholds.

    python tools/fuzz_gpu.py [seconds] [first_seed]

Error metric as in tests/test_gpu_parity.py: ||got - ref|| <= 1e-5 * max(||ref||,
1e-2 ||value of the |.|-network||).  Prints one line per case, FAIL lines with
everything needed to reproduce; exit code 1 on any failure.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness import generators as gen
from paper_2002_01935_b200.harness.paths import greedy_tree
from paper_2002_01935_b200.refpkg import TensorNode
from paper_2002_01935_b200.slicing import greedy_slice
from paper_2002_01935_b200.refpkg import metrics


def make(seed):
    rng = np.random.default_rng(seed)
    kind = seed % 4
    if kind == 3:  # diagonal-reduced circuit: hyperedge-heavy (batched GEMM / SIMT)
        rows, cols = int(rng.integers(4, 7)), int(rng.integers(5, 8))
        tn = gen.grid_circuit(rows, cols, int(rng.integers(10, 25)), seed=seed, diag=True)
    elif kind == 0:
        n = int(rng.integers(60, 140)) // 2 * 2
        tn = gen.random_regular(n, int(rng.choice([3, 4])), seed=seed)
    elif kind == 1:
        rows, cols = int(rng.integers(4, 7)), int(rng.integers(5, 7))
        tn = gen.grid_circuit(rows, cols, int(rng.integers(10, 21)), seed=seed)
    else:
        tn = gen.random_hyper_network(int(rng.integers(18, 30)), int(rng.integers(30, 55)), seed,
                                      max_rank=5, dims=(2, 3, 4))
    tree = greedy_tree(tn, seed=seed, temperature=float(rng.choice([0.0, 0.3])))
    return tn, tree, rng


def abs_value(tn, tree, S, ids):
    atn = tn.replace(nodes=[TensorNode(nd.id, nd.indices, np.abs(nd.data)) for nd in tn.nodes])
    v, _, _ = oracle.contract_sliced(atn, tree, S, slice_ids=ids)
    return float(np.linalg.norm(np.asarray(v).ravel()))


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    t0 = time.time()
    fails = 0
    cases = 0
    kinds = {}
    while time.time() - t0 < budget:
        seed += 1
        tn, tree, rng = make(seed)
        m = metrics(tree, tn)
        if m.width > 24 or m.width < 14:
            continue
        ws = m.width - int(rng.integers(0, 4))
        try:
            ss = greedy_slice(tree, tn, ws, restarts=1, seed=seed) if ws < m.width else ()
        except ValueError:
            ss = ()
        S = tuple(ss.labels) if ss else ()
        prec = str(rng.choice(["3xtf32", "3xtf32", "fp32"]))
        direct = bool(rng.integers(0, 2))
        gmin = float(2 ** int(rng.integers(10, 23)))
        try:
            plan = SlicedPlan(tn, tree, ss, precision=prec, direct_planes=direct, gemm_min_macs=gmin)
        except ValueError as exc:
            print(f"seed {seed}: plan refused ({exc})")
            continue
        d = plan.d
        s1 = min(d, int(rng.integers(1, 5)))
        ids = list(range(s1))
        plan.bind()
        plan.run(0, s1)
        got = np.asarray(plan.result())
        vk = [v["kind"] for v in plan.vertex_info()]
        plan.close()
        ref, _, _ = oracle.contract_sliced(tn, tree, S, slice_ids=ids)
        ref = np.asarray(ref)
        err = float(np.linalg.norm((got - ref).ravel()))
        nref = float(np.linalg.norm(ref.ravel()))
        absv = abs_value(tn, tree, S, ids)
        scale = max(nref, 1e-2 * absv)
        ok = err <= 1e-5 * scale if scale > 0 else err == 0.0
        scale = scale if scale > 0 else 1.0
        cases += 1
        for k in set(vk):
            kinds[k] = kinds.get(k, 0) + 1
        tag = "ok  " if ok else "FAIL"
        print(f"{tag} seed {seed} W={m.width:.1f} Ws={ws} |S|={len(S)} slices={s1} prec={prec} direct={direct} "
              f"gemm_min=2^{int(np.log2(gmin))} gemms={vk.count('gemm_tc')} rel={err / scale:.2e} "
              f"rel_ref={err / nref if nref else 0.0:.2e} abs/ref={absv / nref if nref else 0.0:.1e}", flush=True)
        if not ok:
            fails += 1
    print(f"{cases} cases, {fails} failures; vertex kinds seen: {kinds}")
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
