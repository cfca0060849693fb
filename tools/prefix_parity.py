"""Per-slice and summed error of the GPU executor against the committed oracle
fixtures (tests/golden/northstar_fixtures.json) for one precision setting.

    TNX_GEMM_PROMOTE=1 TNX_GEMM_FIRST=1 python tools/prefix_parity.py d40 [--precision 3xtf32]

Prints one JSON line: per-slice relative error |g - r| / |r|, the slice's
condition ||x_root|| ||y_root|| / |r|, the relative error of the sum over the
fixture's slices, and the slice time.
"""
import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2002_01935_b200.executor import SlicedPlan  # noqa: E402
from paper_2002_01935_b200.harness.workloads import load_workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("key")
    ap.add_argument("--precision", default="3xtf32")
    ap.add_argument("--direct", type=int, default=1)
    ap.add_argument("--raw", default=None, help="no fixture: WORKLOAD:WS:S0-S1, print raw GPU values")
    args = ap.parse_args()
    if args.raw:
        name, ws, rng = args.raw.split(":")
        s0, s1 = (int(x) for x in rng.split("-"))
        tn, tree, ss, _ = load_workload(name, ws=float(ws))
        plan = SlicedPlan(tn, tree, ss, precision=args.precision, direct_planes=bool(args.direct)).bind()
        vals = []
        for s in range(s0, s1):
            plan.reset()
            plan.run(s, s + 1)
            g = complex(plan.result())
            vals.append([s, g.real, g.imag])
        plan.close()
        print(json.dumps({"raw": args.raw, "precision": args.precision, "labels": list(ss.labels),
                          "env": {k: v for k, v in os.environ.items() if k.startswith("TNX_")}, "values": vals}))
        return
    with open(os.path.join(REPO, "tests", "golden", "northstar_fixtures.json")) as fh:
        fx = json.load(fh)[args.key]
    tn, tree, ss, _ = load_workload(fx["workload"], ws=fx["ws"])
    assert list(ss.labels) == fx["sliced_labels"], "slice set differs from the fixture"
    plan = SlicedPlan(tn, tree, ss, precision=args.precision, direct_planes=bool(args.direct)).bind()
    rows, tot_g, tot_r = [], 0j, 0j
    t0 = time.perf_counter()
    for row in fx["slices"]:
        s = row["slice"]
        plan.reset()
        plan.run(s, s + 1)
        g = complex(plan.result())
        r = complex(*row["value"])
        tot_g += g
        tot_r += r
        rows.append({"slice": s, "rel": abs(g - r) / abs(r) if r else None,
                     "bias": ((g - r) * r.conjugate()).real / abs(r) ** 2 if r else None,
                     "cond": row["scale"] / abs(r) if r else None,
                     "normwise": abs(g - r) / row["scale"] if row["scale"] else None})
    dt = time.perf_counter() - t0
    plan.close()
    big = max(abs(complex(*row["value"])) for row in fx["slices"])
    nz = [x for x, row in zip(rows, fx["slices"]) if abs(complex(*row["value"])) > 1e-10 * big]
    rows = [dict(x, zero=abs(complex(*row["value"])) <= 1e-10 * big) for x, row in zip(rows, fx["slices"])]
    rels = [x["rel"] for x in nz]
    out = {"key": args.key, "precision": args.precision,
           "env": {k: v for k, v in os.environ.items() if k.startswith("TNX_")},
           "n": len(rows), "n_nonzero": len(nz), "max_rel": max(rels), "median_rel": sorted(rels)[len(rels) // 2],
           "mean_bias": sum(x["bias"] for x in nz) / len(nz),
           "sum_rel": abs(tot_g - tot_r) / abs(tot_r), "fixture_sum_rel_vs_stored":
           abs(tot_r - complex(*fx["sum"])) / abs(complex(*fx["sum"])),
           "s_per_slice": dt / len(rows), "slices": rows}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
