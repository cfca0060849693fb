"""Hoisted variant of run_perm.py: x has 27 dim-2 labels (2^27 elements) with
interleaved free / contracted labels and is not sliced, so its permute into the
GEMM planes runs once at bind (time it from an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
from paper_2002_01935_b200.refpkg import ContractionTree
rng = np.random.default_rng(0)
ml = [f"m{i}" for i in range(14)]
kl = [f"k{i}" for i in range(13)]
nl = [f"n{i}" for i in range(8)]
xl = [l for pair in zip(ml, kl) for l in pair] + ml[13:]     # interleaved m/k labels
yl = kl[::-1] + nl
tab = {l: 2 for l in ml + kl + nl}
x = np.ones((2,) * len(xl), dtype=np.complex64) * (1 + 0.5j)
y = (rng.standard_normal((2,) * len(yl)) + 0j).astype(np.complex64)
tn = TensorNetwork([TensorNode(0, xl, x), TensorNode(1, yl, y)], tab, tuple(ml + nl))
tree = ContractionTree((0, 1), [(0, 1)])
plan = SlicedPlan(tn, tree, ()).bind()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    prof = plan.profile_slice(0, with_bytes=True)
for k, v, t, b in prof:
    if k == "pack":
        print(f"perm/pack {t:.3f} ms  {b / 1e9:.2f} GB algorithmic  {b / (t / 1e3) / 1e9:.0f} GB/s")
plan.close()
