"""Full-contraction (dot) bandwidth: the library's dot_kernel on two 2^27-element
complex64 operands in the same layout vs torch's cuBLAS complex dot and a plain
read-only reduction, CUDA events, best of 5."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
from paper_2002_01935_b200.refpkg import ContractionTree
n_lab = 26
labels = [f"a{i}" for i in range(n_lab)]
rng = np.random.default_rng(0)
x = (rng.standard_normal(2 ** n_lab) + 1j * rng.standard_normal(2 ** n_lab)).astype(np.complex64).reshape((2,) * n_lab)
y = (rng.standard_normal(2 ** n_lab) + 1j * rng.standard_normal(2 ** n_lab)).astype(np.complex64).reshape((2,) * n_lab)
tn = TensorNetwork([TensorNode(0, labels + ["s"], np.stack([x, x], -1)), TensorNode(1, labels + ["s"], np.stack([y, y], -1))],
                   {**{l: 2 for l in labels}, "s": 2}, ())
plan = SlicedPlan(tn, ContractionTree((0, 1), [(0, 1)]), ("s",)).bind()
best = min(min(t for k, v, t in plan.profile_slice(0) if k == "simt") for _ in range(5))
nbytes = 16 * 2 ** n_lab
print(f"library dot: {best * 1e3:.1f} us  {nbytes / (best / 1e3) / 1e9:.0f} GB/s  kinds {[v['kind'] for v in plan.vertex_info()]}")
plan.close()
xt = torch.from_numpy(x.ravel()).cuda(); yt = torch.from_numpy(y.ravel()).cuda()
def tm(fn):
    b = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); b = min(b, e0.elapsed_time(e1))
    return b
t1 = tm(lambda: torch.dot(xt, yt)); print(f"torch.dot (cuBLAS): {t1 * 1e3:.1f} us  {nbytes / (t1 / 1e3) / 1e9:.0f} GB/s")
xr = torch.view_as_real(xt)
# permuted layouts: y's labels reversed -> fused permute + dot (mode-5 permute kernel)
tnp = TensorNetwork([TensorNode(0, labels + ["s"], np.stack([x, x], -1)),
                     TensorNode(1, labels[::-1] + ["s"], np.stack([y.transpose(), y.transpose()], -1))],
                    {**{l: 2 for l in labels}, "s": 2}, ())
plan = SlicedPlan(tnp, ContractionTree((0, 1), [(0, 1)]), ("s",)).bind()
best = min(min(t for k, v, t in plan.profile_slice(0) if k == "simt") for _ in range(5))
print(f"library perm-dot (y labels reversed): {best * 1e3:.1f} us  {nbytes / (best / 1e3) / 1e9:.0f} GB/s")
plan.close()
t2 = tm(lambda: xr.sum()); print(f"torch.sum (read-only 8 B/elem): {t2 * 1e3:.1f} us  {nbytes / 2 / (t2 / 1e3) / 1e9:.0f} GB/s")
