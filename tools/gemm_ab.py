"""Per-vertex GEMM times of one cfg4 slice (profile_slice, best of 3) for the
current process's GEMM configuration env (e.g. TNX_GEMM_MODEL=0/1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness.workloads import load_workload
tn, tree, ss, _ = load_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg4_7x7_d40", ws=int(sys.argv[2]) if len(sys.argv) > 2 else 27)
plan = SlicedPlan(tn, tree, ss).bind()
info = {v["ssa"]: v for v in plan.vertex_info()}
best = {}
for _ in range(3):
    for k, v, t in plan.profile_slice(0):
        if k == "gemm":
            best[v] = min(best.get(v, 1e9), t)
tot = 0
for v, t in sorted(best.items(), key=lambda x: -x[1]):
    i = info[v]
    fl = 8 * i["m"] * i["n"] * i["k"] * i["batch"]
    tot += t
    print(f"v{v} B={i['batch']} M={i['m']} N={i['n']} K={i['k']} {t:.3f} ms {fl / t / 1e9:.1f} TF/s")
print("gemm total ms", round(tot, 3))
plan.close()
