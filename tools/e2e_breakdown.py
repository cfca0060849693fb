"""Break an e2e bench step (bind from pinned host leaves -> one slice -> D2H)
into its parts on cfg4, with and without slice-invariant hoisting."""
import sys, time
sys.path.insert(0, "."); import numpy as np, torch
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness.workloads import load_workload
tn, tree, ss, _ = load_workload("cfg4_7x7_d40", ws=27)
hoist = not (len(sys.argv) > 1 and sys.argv[1] == "nohoist")
plan = SlicedPlan(tn, tree, ss, hoist=hoist).bind()
leaves = [torch.from_numpy(np.ascontiguousarray(tn.node(n).data, dtype=np.complex128)).pin_memory().numpy() for n in tree.leaves]
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
for _ in range(3):
    plan.bind(leaf_arrays=leaves, stream=s); plan.run(0, 1, s); plan.result(s)
torch.cuda.synchronize()
tb, tr, tres = [], [], []
for i in range(10):
    t0 = time.perf_counter(); plan.bind(leaf_arrays=leaves, stream=s); torch.cuda.synchronize(); t1 = time.perf_counter()
    plan.run(i, i + 1, s); torch.cuda.synchronize(); t2 = time.perf_counter()
    plan.result(s); t3 = time.perf_counter()
    tb.append(t1 - t0); tr.append(t2 - t1); tres.append(t3 - t2)
print(("hoist " if hoist else "nohoist ") + "bind %.3f ms  slice %.3f ms  result %.3f ms" % (1e3 * np.median(tb), 1e3 * np.median(tr), 1e3 * np.median(tres)))
