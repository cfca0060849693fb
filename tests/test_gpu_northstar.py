"""North-star parity (BASELINE.json north_star):
the sliced 7x7 (1+40+1) circuit amplitude workload, the full 7x7 (1+24+1)
amplitude and 8 slices of the Sycamore-53 m=12 amplitude (configs[4]), GPU (default precision: split-TF32 tensor cores + FP32 SIMT,
complex64 storage) against complex128 oracle values.

The oracle needs ~20 s per d40 slice on 16 cores, so its values are committed
fixtures (tests/golden/northstar_fixtures.json, made by
tests/golden/make_circuit_fixtures.py from the same seeded networks, trees and
slice sets).  Tolerance, written here: PLAIN relative error
|c_gpu - c_ref| / |c_ref| <= 1e-5 for every slice that is not zero in exact
arithmetic, for the sum over the fixture's slices, and for the full d24
amplitude.  Slices that are exactly zero in exact arithmetic (about half of
this circuit's slices: a sliced CZ bond projects a |0> input onto |1>) come out
of the complex128 oracle as ~1e-16 of the nonzero slices' magnitude and have no
relative error (the GPU's complex64 round-off of them is ~1e-8 of the nonzero
slices, the oracle's complex128 one ~1e-16); for them the test asserts |c_gpu|
stays below 1e-7 of the largest slice of the set.  Each slice's condition ||x_root|| ||y_root|| / |c|
is printed beside its error.
"""
import json
import os

import numpy as np
import pytest

from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.harness.workloads import load_workload

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "northstar_fixtures.json")) as _fh:
    FIX = json.load(_fh)

TOL = 1e-5


def _run(key):
    fx = FIX[key]
    tn, tree, ss, meta = load_workload(fx["workload"], ws=fx["ws"])
    assert list(ss.labels) == fx["sliced_labels"], "slicer output differs from the fixture's"
    assert int(ss.d) == fx["d"]
    plan = SlicedPlan(tn, tree, ss).bind()
    try:
        assert plan.stats()["num_gemm"] > 0
        assert plan.ops_per_slice == fx["ops_per_slice"]
        got = []
        for row in fx["slices"]:
            s = row["slice"]
            plan.reset()
            plan.run(s, s + 1)
            got.append(complex(plan.result()))
        if fx["complete"]:
            plan.reset()
            plan.run()
            total = complex(plan.result())
        else:
            total = None
    finally:
        plan.close()
    return fx, got, total


@pytest.mark.parametrize("key", ["d40", "d40r", "d40g", "d40gr", "d24", "syc"])
def test_northstar_slices(key):
    if key not in FIX:
        pytest.fail(f"fixture {key} missing: run tests/golden/make_circuit_fixtures.py {key}")
    fx, got, total = _run(key)
    refs = [complex(*r["value"]) for r in fx["slices"]]
    big = max(abs(r) for r in refs)
    lines, worst = [], 0.0
    for row, g, r in zip(fx["slices"], got, refs):
        if abs(r) <= 1e-10 * big:  # zero in exact arithmetic
            assert abs(g) <= 1e-7 * big, (row["slice"], g, r)
            lines.append(f"slice {row['slice']}: exact zero (|gpu| {abs(g) / big:.1e} of max)")
            continue
        rel = abs(g - r) / abs(r)
        worst = max(worst, rel)
        lines.append(f"slice {row['slice']}: rel {rel:.2e} cond {row['scale'] / abs(r):.1e}")
    print(f"\n{key} ({fx['workload']}, W_s={fx['ws']}): worst slice rel {worst:.2e}\n  " + "\n  ".join(lines))
    assert worst <= TOL, lines
    sg, sr = sum(got), sum(refs)
    assert abs(sg - sr) <= TOL * abs(sr), (sg, sr, abs(sg - sr) / abs(sr))
    if total is not None:
        # full amplitude through the public accumulate path (Kahan, complex128)
        ref_total = complex(*fx["sum"])
        err = abs(total - ref_total) / abs(ref_total)
        print(f"  full amplitude over {fx['d']} slices: rel {err:.2e}")
        assert err <= TOL, (total, ref_total, err)
        assert np.isclose(sr, ref_total, rtol=1e-12, atol=0)
