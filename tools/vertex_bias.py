"""Local error of every GEMM vertex of one slice on real workload data.

    python tools/vertex_bias.py [config] [slice] [ws]

For each tensor-core vertex v (and the root) the GPU result (tnx_debug_vertex)
is compared with the complex128 contraction of the GPU's OWN children values,
so the numbers isolate v's own arithmetic error from what it inherited:
  rel  = ||z_gpu - z_exact|| / ||z_exact||
  bias = Re<z_gpu - z_exact, z_exact> / ||z_exact||^2   (< 0: uniform shrink)
  canc = ||x|| ||y|| / ||z_exact||  (cancellation inside the contraction)
Also the accumulated error of v against the oracle's chain (rel_chain).
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2002_01935_b200.executor import SlicedPlan  # noqa: E402
from paper_2002_01935_b200.harness.workloads import load_workload  # noqa: E402
from paper_2002_01935_b200.slicing import slice_assignment  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4_7x7_d40"
    sid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    ws = float(sys.argv[3]) if len(sys.argv) > 3 else None
    tn, tree, ss, meta = load_workload(cfg, ws=ws)
    plan = SlicedPlan(tn, tree, ss, direct_planes=False).bind()
    info = {v["ssa"]: v for v in plan.vertex_info()}
    rec = {}
    t = time.time()
    oracle.contract_one(tn, tree, ss.labels, slice_assignment(tn, ss, sid), record=rec)
    print("oracle slice", sid, "in", round(time.time() - t, 1), "s", flush=True)
    terms = oracle.vertex_terms(tn, tree)
    n = len(tree.leaves)
    asg = slice_assignment(tn, ss, sid)

    def gpu_val(u):
        if u < n:  # leaf: the GPU contracts the complex64 leaf, sliced
            nd = tn.node(tree.leaves[u])
            labels, arr = tuple(nd.indices), nd.data.astype(np.complex64).astype(np.complex128)
            for lbl in ss.labels:
                if lbl in labels:
                    labels, arr = oracle.fix_index(labels, arr, lbl, asg[lbl])
            return labels, arr
        labels, arr = plan.debug_vertex(sid, u)
        return tuple(labels), arr.astype(np.complex128)

    S = set(ss.labels)
    tot_bias = 0.0
    for v in sorted(info):
        x = info[v]
        if x["kind"] != "gemm_tc" and v != tree.root:
            continue
        a, b = tree.children(v)
        xl, xa = gpu_val(a)
        yl, ya = gpu_val(b)
        zl, za = gpu_val(v)
        keep = set(terms[v]) - S
        ol, exact = oracle.pairwise_contract(xl, xa, yl, ya, keep)
        exact = np.transpose(exact, [ol.index(lbl) for lbl in zl]) if zl else exact
        d = (za - exact).ravel()
        e = exact.ravel()
        nrm = np.linalg.norm(e)
        rel = np.linalg.norm(d) / nrm
        bias = np.vdot(e, d).real / nrm ** 2
        canc = np.linalg.norm(xa) * np.linalg.norm(ya) / nrm
        cl, chain = rec[v]
        chain = np.transpose(chain, [cl.index(lbl) for lbl in zl]) if zl else chain
        rc = np.linalg.norm((za - chain).ravel()) / np.linalg.norm(chain.ravel())
        bc = np.vdot(chain.ravel(), (za - chain).ravel()).real / np.linalg.norm(chain.ravel()) ** 2
        tot_bias += bias
        print(f"v={v} {x['kind']:8s} hoisted={x['hoisted']} M={x['m']} N={x['n']} K={x['k']} B={x['batch']} "
              f"rel={rel:.2e} bias={bias:+.2e} canc={canc:.1e} | chain rel={rc:.2e} bias={bc:+.2e}", flush=True)
    print(f"sum of local GEMM biases {tot_bias:+.2e}")
    plan.close()


if __name__ == "__main__":
    main()
