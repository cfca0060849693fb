"""Oracle fixtures for the north-star parity tests (tests/test_gpu_northstar.py).

The CPU oracle needs minutes for these (a cfg4 d40 slice is 8.2e12 flop), so
the values are computed once here and committed as
``tests/golden/northstar_fixtures.json``; the GPU tests regenerate the same
seeded networks, trees and slice sets and compare against the stored values.

    python tests/golden/make_circuit_fixtures.py [d24] [d40] [d40r]

* ``d24``  -- every slice of the 7x7 (1+24+1) amplitude at W_s=27 (32 slices,
  reference min-fill tree): per-slice values and the full amplitude.
* ``d40``  -- the first 16 ids of the bench workload's nonzero-slice list
  (7x7 (1+40+1), W_s=27, reference min-fill tree; benchdata/
  cfg4_7x7_d40.slices.json -- this tree's slices [0, 1024) are all zero in
  exact arithmetic).
* ``d40r`` -- 8 seeded picks from the rest of that list.
* ``d40g`` / ``d40gr`` -- the same for the greedy-driver tree (cfg4g).
* ``syc``  -- slices 0..7 of configs[4] (Sycamore-53 m=12, W_s=27).

Per slice it stores the value, its root-operand scale ||x|| ||y|| (the
condition of the last contraction) and the slice's label assignment digits, so
a change in the generator, tree or slicer is caught as a fixture mismatch
rather than as a numerical failure.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import oracle  # noqa: E402
from paper_2002_01935_b200.harness.workloads import load_workload  # noqa: E402
from paper_2002_01935_b200.slicing import slice_assignment  # noqa: E402

OUT = os.path.join(HERE, "northstar_fixtures.json")

SETS = {
    "d24": ("cfg4p_7x7_d24", 27, "all"),
    "d40": ("cfg4_7x7_d40", 27, "nonzero:0:16"),
    "d40r": ("cfg4_7x7_d40", 27, "nonzero-random8"),
    # the same circuit under the greedy-driver tree (round-1 bench workload)
    "d40g": ("cfg4g_7x7_d40", 27, list(range(16))),
    "d40gr": ("cfg4g_7x7_d40", 27, "random8"),
    # BASELINE configs[4]: Sycamore-like 53-qubit m=12 amplitude (synthetic fSim)
    "syc": ("cfg5_syc53_m12", 27, list(range(8))),
}


def nonzero_ids(name):
    """Slice ids of the workload that are nonzero in exact arithmetic
    (benchdata/<name>.slices.json, found by tools/slice_scan.py)."""
    with open(os.path.join(REPO, "benchdata", f"{name}.slices.json")) as fh:
        return [int(x) for x in json.load(fh)["ids"]]


def slice_ids(spec, d, name=None):
    if spec == "all":
        return list(range(d))
    if isinstance(spec, str) and spec.startswith("nonzero:"):
        a, b = (int(x) for x in spec.split(":")[1:])
        return nonzero_ids(name)[a:b]
    if spec == "nonzero-random8":
        rest = nonzero_ids(name)[16:]
        rng = np.random.default_rng(2002)
        return sorted(int(rest[i]) for i in rng.choice(len(rest), size=8, replace=False))
    if spec == "random8":
        rng = np.random.default_rng(2002)
        return sorted(int(x) for x in rng.integers(0, d, size=8, dtype=np.int64))
    return list(spec)


def run(key):
    name, ws, spec = SETS[key]
    tn, tree, ss, meta = load_workload(name, ws=ws)
    ids = slice_ids(spec, ss.d, name)
    terms = oracle.vertex_terms(tn, tree)
    root = tree.root
    a, b = tree.children(root)
    keep = {a, b}

    class Rec(dict):
        def __setitem__(self, k, v):
            if k in keep:
                dict.__setitem__(self, k, v)

    rows = []
    acc = oracle.oracle._Kahan(())
    t0 = time.time()
    for s in ids:
        rec = Rec()
        asg = slice_assignment(tn, ss, s)
        r, _, ops, _ = oracle.contract_one(tn, tree, ss.labels, asg, terms=terms, record=rec)
        val = complex(np.asarray(r))
        scale = float(np.linalg.norm(rec[a][1].ravel()) * np.linalg.norm(rec[b][1].ravel()))
        acc.add(np.asarray(r))
        rows.append({"slice": s, "value": [val.real, val.imag], "scale": scale,
                     "digits": [int(asg[lbl]) for lbl in ss.labels]})
        print(f"{key} slice {s}: {val:.6e} scale {scale:.3e} ({time.time() - t0:.0f}s)", flush=True)
    total = complex(acc.s)
    return {"workload": name, "ws": ws, "sliced_labels": list(ss.labels), "d": int(ss.d),
            "ops_per_slice": int(ss.per_slice_cost), "tree_W": meta["W"], "tree_log10_C": meta["log10_C"],
            "slices": rows, "sum": [total.real, total.imag], "complete": len(ids) == ss.d,
            "seconds": time.time() - t0}


def main(keys):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    for key in keys:
        data[key] = run(key)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SETS))
