"""SIMT contraction kernels on HBM-bound shapes (K4): (a) skinny, many outputs
x[s, a(20), k(4)] . y[s, k(4)] -> [a] (thread mode, 2^20 outputs x 16 terms);
(b) few outputs, long sums x[s, b(10), j(14)] . y[s, j(14)] -> [b] (warp / split
mode).  Prints per-launch time and algorithmic bytes (x and y read once, output
written once) -> GB/s."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
from paper_2002_01935_b200.refpkg import ContractionTree
rng = np.random.default_rng(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3


def case(outl, sumd, name):
    sl = [f"k{i}" for i in range(sumd)]
    xl, yl = ["s"] + outl + sl, ["s"] + sl
    tab = {l: 2 for l in xl}
    x = (rng.standard_normal([2] * len(xl)) + 0j).astype(np.complex64)
    y = (rng.standard_normal([2] * len(yl)) + 0j).astype(np.complex64)
    tn = TensorNetwork([TensorNode(0, xl, x), TensorNode(1, yl, y)], tab, tuple(outl))
    plan = SlicedPlan(tn, ContractionTree((0, 1), [(0, 1)]), ("s",)).bind()
    kind = plan.vertex_info()[0]["kind"]
    best = 1e9
    for _ in range(reps):
        best = min(best, min(t for k, v, t in plan.profile_slice(0) if k == "simt"))
    nbytes = 8 * (x.size // 2 + y.size // 2 + 2 ** len(outl))
    print(f"{name}: kind={kind} {best * 1e3:.1f} us  {nbytes / 1e6:.1f} MB algorithmic  "
          f"{nbytes / (best / 1e3) / 1e9:.0f} GB/s")
    plan.close()


case([f"a{i}" for i in range(20)], 4, "skinny (2^20 outputs x 16)")
case([f"b{i}" for i in range(10)], 14, "long sums (2^10 outputs x 2^14)")
