"""Time the tcgen05 GEMM kernel alone (CUDA events around the kernel via a
pre-packed plan) and its error for a few shapes.  Env TNX_GEMM_PROMOTE set by caller."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
# two-tensor network whose single vertex is a GEMM: x[m..,k..], y[n..,k..]
def net(lm, ln, lk, seed):
    rng = np.random.default_rng(seed)
    ml = [f"m{i}" for i in range(lm)]; nl = [f"n{i}" for i in range(ln)]; kl = [f"k{i}" for i in range(lk)]
    tab = {l: 2 for l in ml + nl + kl}
    x = (rng.standard_normal((2,)*(lm+lk)) + 1j*rng.standard_normal((2,)*(lm+lk)))
    y = (rng.standard_normal((2,)*(ln+lk)) + 1j*rng.standard_normal((2,)*(ln+lk)))
    return TensorNetwork([TensorNode(0, ml+kl, x), TensorNode(1, nl+kl, y)], tab, tuple(ml+nl))
from paper_2002_01935_b200.refpkg import ContractionTree
for (lm, ln, lk) in [(13, 13, 12), (12, 12, 14), (11, 11, 16)]:
    tn = net(lm, ln, lk, 0)
    tree = ContractionTree((0, 1), [(0, 1)])
    plan = SlicedPlan(tn, tree, (), precision=os.environ.get('PREC', '3xtf32')).bind()
    g = [min(t for k, v, t in plan.profile_slice(0) if k == "gemm") for _ in range(4)]
    g = [min(g)]
    plan.run(); val = plan.result()
    x = tn.node(0).data.reshape(2**lm, 2**lk); y = tn.node(1).data.reshape(2**ln, 2**lk)
    ref = (x @ y.T).reshape(val.shape)
    err = np.linalg.norm(val - ref) / np.linalg.norm(ref)
    fl = 8 * 2**(lm+ln+lk)
    print(f"prec={os.environ.get('PREC','3xtf32')} M=2^{lm} N=2^{ln} K=2^{lk}: gemm {g[0]:.3f} ms "
          f"{fl/g[0]/1e9:.1f} TF/s  rel_err {err:.2e}", flush=True)
    plan.close()
