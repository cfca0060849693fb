"""Small-K GEMM fused into its parent (the shape of cfg4 vertex 1463:
M=4096, N=8192, K=8, output written straight into the parent's split-TF32
planes).  child = x[s, a(12), k(3)] . y[k(3), b(13)]; parent = child . w[s, b, c(8)]
(s sliced, so both run per slice).  Prints per-launch times of one slice."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
from paper_2002_01935_b200.refpkg import ContractionTree
rng = np.random.default_rng(0)
# optional label counts: run_smallk.py reps [n_a n_k n_b n_c]  (M = 2^n_a, K = 2^n_k, N = 2^n_b)
na, nk, nb, nc = (int(x) for x in sys.argv[2:6]) if len(sys.argv) > 5 else (12, 3, 13, 8)
al = [f"a{i}" for i in range(na)]
kl = [f"k{i}" for i in range(nk)]
bl = [f"b{i}" for i in range(nb)]
cl = [f"c{i}" for i in range(nc)]
tab = {l: 2 for l in al + kl + bl + cl + ["s"]}
def rnd(ls):
    shp = [tab[l] for l in ls]
    return ((rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / 4).astype(np.complex64)
x, y, w = rnd(["s"] + al + kl), rnd(kl + bl), rnd(["s"] + bl + cl)
tn = TensorNetwork([TensorNode(0, ["s"] + al + kl, x), TensorNode(1, kl + bl, y),
                    TensorNode(2, ["s"] + bl + cl, w)], tab, tuple(al + cl))
tree = ContractionTree((0, 1, 2), [(0, 1), (3, 2)])
plan = SlicedPlan(tn, tree, ("s",)).bind()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
best = {}
for _ in range(reps):
    for k, v, t in plan.profile_slice(0):
        best[(k, v)] = min(best.get((k, v), 1e9), t)
info = {v["ssa"]: v for v in plan.vertex_info()}
for (k, v), t in best.items():
    extra = ""
    if k == "gemm":
        i = info[v]
        extra = f"M={i['m']} N={i['n']} K={i['k']}  out {i['m'] * i['n'] / 1e6:.1f}M elems"
    print(k, v, f"{t:.4f} ms", extra)
plan.close()
