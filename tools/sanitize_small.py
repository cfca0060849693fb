"""Small workload touching every kernel (gather, batched SIMT, perm, pack,
1-CTA and 2-CTA GEMM, direct planes, split-K, dot, accum) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness.workloads import load_workload
from paper_2002_01935_b200.harness import generators as gen

tn, tree, ss, _ = load_workload("cfg4p_7x7_d20", ws=24)
plan = SlicedPlan(tn, tree, ss, gemm_min_macs=2 ** 12, graph=False).bind()
kinds = sorted({v["kind"] for v in plan.vertex_info()})
plan.run(0, 2)
v1 = plan.result()
plan.close()
ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels, slice_ids=range(0, 2))
print("kinds", kinds, "rel", abs(complex(v1) - ref) / abs(ref))
tn = gen.random_hyper_network(8, 14, seed=101, max_rank=5)
from paper_2002_01935_b200.harness.paths import greedy_tree
t2 = greedy_tree(tn)
p2 = SlicedPlan(tn, t2, [l for l in tn.index_table if l not in tn.output][:2], graph=False).bind()
p2.run()
print("hyper ok", np.asarray(p2.result()).shape)
p2.close()
