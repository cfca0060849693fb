"""Per-launch profile of one slice of a workload (best of 3): non-GEMM
launches with algorithmic bytes and achieved GB/s, plus totals by kind."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness.workloads import load_workload
tn, tree, ss, _ = load_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg4_7x7_d40",
                                ws=int(sys.argv[2]) if len(sys.argv) > 2 else 27)
plan = SlicedPlan(tn, tree, ss).bind()
best = None
for _ in range(3):
    prof = plan.profile_slice(0, with_bytes=True)
    if best is None:
        best = [list(p) for p in prof]
    else:
        for b, p in zip(best, prof):
            b[2] = min(b[2], p[2])
tot = {}
for k, v, t, b in best:
    tot[k] = tot.get(k, 0) + t
    if k != "gemm" and t > 0.004:
        print(f"{k:6s} v{v:5d} {t * 1e3:8.1f} us  {b / 1e6:8.2f} MB  {b / (t / 1e3) / 1e9 if t else 0:8.0f} GB/s")
print({k: round(t, 3) for k, t in tot.items()}, "launches", len(best))
plan.close()
