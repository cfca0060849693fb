"""Per-vertex parity of one slice of a benchmark workload: every slice-
dependent intermediate from the GPU (tnx_debug_vertex) vs the CPU oracle
(complex128), norm-wise.  Usage: python tools/parity_slice.py [config] [slice] [ws]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2002_01935_b200.harness.workloads import load_workload
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.slicing import slice_assignment

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4_7x7_d40"
sid = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ws = float(sys.argv[3]) if len(sys.argv) > 3 else None
tn, tree, ss, meta = load_workload(cfg, ws=ws)
plan = SlicedPlan(tn, tree, ss, direct_planes=False).bind()  # precision from TNX_PRECISION
info = {v["ssa"]: v for v in plan.vertex_info()}
rec = {}
t = time.time()
oracle.contract_one(tn, tree, ss.labels, slice_assignment(tn, ss, sid), record=rec)
print("oracle slice", sid, "in", round(time.time() - t, 1), "s")
worst = 0.0
for v in sorted(info):
    x = info[v]
    if x["hoisted"]:
        continue
    labels, arr = plan.debug_vertex(sid, v)
    ol, oarr = rec[v]
    oarr = np.transpose(oarr, [ol.index(l) for l in labels]) if labels else oarr
    nrm = np.linalg.norm(oarr.ravel())
    a, b = tree.children(v)
    na = np.linalg.norm(rec[a][1].ravel()) if a in rec else np.linalg.norm(tn.node(tree.leaves[a]).data.ravel())
    nb = np.linalg.norm(rec[b][1].ravel()) if b in rec else np.linalg.norm(tn.node(tree.leaves[b]).data.ravel())
    diff = np.linalg.norm((arr.astype(np.complex128) - oarr).ravel())
    err = diff / (na * nb)           # normwise vs the operand scale
    rel = diff / nrm if nrm > 0 else float("inf")
    worst = max(worst, err)
    if x["kind"] == "gemm_tc" or err > 1e-6 or x["rank"] == 0:
        print(f"v={v} {x['kind']:12s} rank={x['rank']:2d} M={x['m']} N={x['n']} K={x['k']} "
              f"|ref|={nrm:.3e} |x||y|={na*nb:.3e} err/(|x||y|)={err:.2e} rel={rel:.2e}")
print("worst ||dz||/(||x|| ||y||) over dependent vertices:", worst)
plan.close()
