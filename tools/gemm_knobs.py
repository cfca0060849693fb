"""Standalone tcgen05 GEMM time and per-clock efficiency for given shapes
(A/B of the TNX_GEMM_* knobs, set by the caller).

    TNX_GEMM_FIRST=12 python tools/gemm_knobs.py 8192x16384x512 32768x4096x512

Each shape is a two-tensor network (x[m,k] y[n,k], dims 2) whose single vertex
is a GEMM; the kernel time comes from tnx_profile_slice (CUDA events around
the launch), the SM clock from clock64/globaltimer stamps around a few graph
replays of the same plan (the GEMM is >95 % of each replay).  Efficiency =
8 M N K * 3 / (148 SMs * clock * time) / 4080 flop/clk/SM (tnx_mma_peak).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_01935_b200 import _native  # noqa: E402
from paper_2002_01935_b200.executor import SlicedPlan  # noqa: E402
from paper_2002_01935_b200.refpkg import ContractionTree, TensorNetwork, TensorNode  # noqa: E402


def net(lm, ln, lk, seed=0, lq=0):
    """x[m,k] y[n,k] (-> z[m,n]); with lq > 0 also w[n,q], so z feeds a GEMM
    parent contracting n and the measured GEMM writes the parent's operand
    planes (the direct-plane epilogue the tree's inner GEMMs use)."""
    rng = np.random.default_rng(seed)
    ml = [f"m{i}" for i in range(lm)]
    nl = [f"n{i}" for i in range(ln)]
    kl = [f"k{i}" for i in range(lk)]
    ql = [f"q{i}" for i in range(lq)]
    tab = {lbl: 2 for lbl in ml + nl + kl + ql}
    x = rng.standard_normal((2,) * (lm + lk)) + 1j * rng.standard_normal((2,) * (lm + lk))
    y = rng.standard_normal((2,) * (ln + lk)) + 1j * rng.standard_normal((2,) * (ln + lk))
    nodes = [TensorNode(0, ml + kl, x), TensorNode(1, nl + kl, y)]
    if lq:
        w = rng.standard_normal((2,) * (ln + lq)) + 1j * rng.standard_normal((2,) * (ln + lq))
        nodes.append(TensorNode(2, nl + ql, w))
        return TensorNetwork(nodes, tab, tuple(ml + ql))
    return TensorNetwork(nodes, tab, tuple(ml + nl))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--chain=")]
    lq = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--chain=")), 0))
    shapes = [tuple(int(v) for v in a.split("x")) for a in args] or [(8192, 16384, 512)]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for M, N, K in shapes:
        lm, ln, lk = (int(np.log2(v)) for v in (M, N, K))
        tn = net(lm, ln, lk, lq=lq)
        tree = ContractionTree((0, 1, 2), [(0, 1), (3, 2)]) if lq else ContractionTree((0, 1), [(0, 1)])
        plan = SlicedPlan(tn, tree, ()).bind()
        t = min([tt for k, v, tt in plan.profile_slice(0) if k == "gemm" and v == len(tree.leaves)][0]
                for _ in range(3))
        st = torch.cuda.Stream()
        stamps = _native.ClockStamps()
        stamps.start(st.cuda_stream)
        for _ in range(4):
            plan.run(0, 1, st)
        stamps.stop(st.cuda_stream)
        torch.cuda.synchronize()
        mhz, _ = stamps.mhz()
        plan.close()
        fl = 8.0 * M * N * K
        eff = fl * 3 / (sms * mhz * 1e6 * t * 1e-3) / 4080.0
        print(json.dumps({"M": M, "N": N, "K": K, "chain_q": lq, "ms": t, "tflops": fl / t / 1e9, "mhz": mhz, "eff_per_clk": eff,
                          "env": {k: v for k, v in os.environ.items() if k.startswith("TNX_")}}), flush=True)


if __name__ == "__main__":
    main()
