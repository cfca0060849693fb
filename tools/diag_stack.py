import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import oracle
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness import generators as gen
from paper_2002_01935_b200.harness.paths import best_greedy_tree
from paper_2002_01935_b200.slicing import greedy_slice
from paper_2002_01935_b200.tree import metrics
from _util import rel_err
tn = gen.grid_circuit(5, 5, 24, seed=7)
tree = best_greedy_tree(tn, trials=3)
m = metrics(tree, tn)
ss = greedy_slice(tree, tn, min(m.width, 23) - 1, restarts=1)
ref, _, _ = oracle.contract_sliced(tn, tree, ss.labels, slice_ids=range(0, min(ss.d, 4)))
for tiled in (True, False):
    for direct in (True, False):
        plan = SlicedPlan(tn, tree, ss, gemm_min_macs=2 ** 14, tiled_pack=tiled, direct_planes=direct).bind()
        plan.run(0, min(plan.d, 4))
        print("tiled", tiled, "direct", direct, rel_err(plan.result(), ref), plan.stats()["num_gemm"])
        plan.close()
