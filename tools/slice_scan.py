"""Per-slice magnitudes of a workload on the GPU: which slices are zero in
exact arithmetic (they come out as complex64 round-off, ~1e-7 or less of the
nonzero slices) and which carry the amplitude.

    python tools/slice_scan.py cfg4_7x7_d40 27 1024 [--random 1024]

Prints one JSON line: the magnitudes of slices [0, N) and of a seeded random
sample of slice ids, and the ids whose magnitude is within 1e-4 of the
largest seen (the nonzero ones).
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from paper_2002_01935_b200.executor import SlicedPlan  # noqa: E402
from paper_2002_01935_b200.harness.workloads import load_workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("ws", type=float)
    ap.add_argument("n", type=int)
    ap.add_argument("--random", type=int, default=0)
    args = ap.parse_args()
    tn, tree, ss, _ = load_workload(args.workload, ws=args.ws)
    plan = SlicedPlan(tn, tree, ss).bind()
    rng = np.random.default_rng(7)
    ids = list(range(args.n)) + sorted(int(x) for x in rng.integers(0, ss.d, size=args.random, dtype=np.int64))
    mags = []
    for s in ids:
        plan.reset()
        plan.run(s, s + 1)
        mags.append(abs(complex(plan.result())))
    plan.close()
    big = max(mags)
    nonzero = [s for s, m in zip(ids, mags) if m >= 1e-4 * big]
    print(json.dumps({"workload": args.workload, "ws": args.ws, "d": str(ss.d), "ids": ids, "mags": mags,
                      "max": big, "nonzero": nonzero,
                      "nonzero_prefix": sum(1 for s in nonzero if s < args.n) / max(1, args.n),
                      "nonzero_random": sum(1 for s in nonzero if s >= args.n) / max(1, args.random)}))


if __name__ == "__main__":
    main()
