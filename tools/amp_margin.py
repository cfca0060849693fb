"""Relative error of full sliced amplitudes (7x7 d16/d20) vs the complex128
oracle, per precision mode (env TNX_PRECISION / TNX_GEMM_PROMOTE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness.workloads import load_workload
for name, ws in (("cfg4p_7x7_d16", 16), ("cfg4p_7x7_d20", 24), ("cfg4p_7x7_d20", 21)):
    tn, tree, ss, _ = load_workload(name, ws=ws)
    ref, _, _ = oracle.contract(tn, tree)
    for prec in os.environ.get("PRECS", "3xtf32,tf32-bf16x,fp32").split(","):
        plan = SlicedPlan(tn, tree, ss, precision=prec).bind()
        plan.run()
        got = complex(plan.result())
        plan.close()
        print(f"{name} ws={ws} {prec:11s} promote={os.environ.get('TNX_GEMM_PROMOTE', '3 (default)')} "
              f"rel_err={abs(got - ref) / abs(ref):.3e}", flush=True)
