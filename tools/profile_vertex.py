"""Profile one tensor-core vertex of a workload slice with ncu.

    python tools/profile_vertex.py cfg5_syc53_m12 417            # prints the launch index
    ncu --nvtx --nvtx-include "slice/" -k regex:gemm_c64 --launch-skip I -c 1 ... \\
        python tools/profile_vertex.py cfg5_syc53_m12 417

Binds the workload's plan (hoisted kernels run outside the NVTX range), then
runs one slice launch by launch (tnx_profile_slice) inside the NVTX range
"slice"; I is the position of vertex V among that slice's GEMM launches.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2002_01935_b200.executor import SlicedPlan  # noqa: E402
from paper_2002_01935_b200.harness.workloads import load_workload  # noqa: E402


def main():
    name, v = sys.argv[1], int(sys.argv[2])
    tn, tree, ss, _ = load_workload(name)
    plan = SlicedPlan(tn, tree, ss).bind()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("slice")
    prof = plan.profile_slice(0)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    gemms = [vv for k, vv, t in prof if k == "gemm"]
    info = {x["ssa"]: x for x in plan.vertex_info()}
    x = info[v]
    t = [tt for k, vv, tt in prof if vv == v and k == "gemm"][0]
    print(f"vertex {v} M={x['m']} N={x['n']} K={x['k']} batch={x['batch']}: gemm launch index {gemms.index(v)} "
          f"of {len(gemms)}; {t:.3f} ms, {8 * x['macs'] / t / 1e9:.1f} TFLOP/s")
    plan.close()


if __name__ == "__main__":
    main()
