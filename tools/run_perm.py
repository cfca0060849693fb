"""Large operand permute (K2) feeding a GEMM: x has 13 dim-4 labels (+ a sliced dim-2 label) in an order
that interleaves free and contracted labels, so packing it into the GEMM's
K-blocked split-TF32 planes is a genuine transpose.  Prints the perm launch
time and its algorithmic HBM bandwidth (8 B read + 16 B written per element)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
from paper_2002_01935_b200.refpkg import ContractionTree
rng = np.random.default_rng(0)
ml = [f"m{i}" for i in range(7)]   # dim 4 labels: x slice = 4^13 = 2^26 elements
kl = [f"k{i}" for i in range(6)]
nl = [f"n{i}" for i in range(4)]
xl = ["s"] + [l for pair in zip(ml, kl) for l in pair] + ml[6:]  # interleaved m/k labels
yl = ["s"] + kl[::-1] + nl
tab = {l: 4 for l in ml + kl + nl}
tab["s"] = 2
x = np.ones([tab[l] for l in xl], dtype=np.complex64) * (1 + 0.5j)
y = (rng.standard_normal([tab[l] for l in yl]) + 0j).astype(np.complex64)
tn = TensorNetwork([TensorNode(0, xl, x), TensorNode(1, yl, y)], tab, tuple(ml + nl))
tree = ContractionTree((0, 1), [(0, 1)])
plan = SlicedPlan(tn, tree, ("s",)).bind()   # sliced: x is re-packed every slice
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    prof = plan.profile_slice(0, with_bytes=True)
for k, v, t, b in prof:
    print(k, v, f"{t:.3f} ms")
    if k == "pack" and t > 0.1:
        print(f"perm/pack {t:.3f} ms  {b / 1e9:.2f} GB algorithmic  {b / (t / 1e3) / 1e9:.0f} GB/s")
plan.close()
