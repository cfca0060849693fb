"""C-ABI library: loads, exports every declared symbol, and its plan
compiler reproduces the reference bookkeeping bit-exactly (no GPU needed:
tnx_plan_create touches no device state)."""
import os
import re

import pytest

from conftest import golden_cases, load_golden, REPO
from _util import case_objects
from paper_2002_01935_b200 import _native as nat
from paper_2002_01935_b200.executor import SlicedPlan
from paper_2002_01935_b200.slicing import sliced_metrics
from paper_2002_01935_b200.refpkg import ContractionTree, metrics
from paper_2002_01935_b200.harness import generators as gen


def test_library_exports_every_header_symbol():
    lib = nat.load()
    hdr = open(os.path.join(REPO, "include", "tnx.h")).read()
    declared = set(re.findall(r"\b(tnx_[a-z_0-9]+)\s*\(", hdr))
    assert declared, "no symbols parsed"
    assert declared == set(nat.SIGNATURES), declared ^ set(nat.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name)
    assert b"sm_100a" in lib.tnx_version()


CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_native_bookkeeping_matches_reference(case):
    tn, tree = case_objects(case)
    for ent in case["sliced"]:
        plan = SlicedPlan(tn, tree, ent["labels"])
        assert plan.d == ent["d"]
        assert plan.ops_per_slice * plan.d == int(ent["Cs"])
        assert plan.width == ent["Ws"]
        plan.close()


STRUCT = load_golden("reference_structural.json")


@pytest.mark.parametrize("case", STRUCT, ids=[c["name"] for c in STRUCT])
def test_native_bookkeeping_big_configs(case):
    tn = {"cfg2_5reg100": lambda: gen.random_regular(100, 5, seed=0),
          "cfg3_lattice20": lambda: gen.square_lattice(20, seed=0),
          "cfg4_7x7_d40": lambda: gen.grid_circuit(7, 7, 40, seed=0)}[case["name"]]()
    tree = ContractionTree(case["tree"]["leaves"], [tuple(p) for p in case["tree"]["pairs"]])
    plan = SlicedPlan(tn, tree, ())
    assert plan.ops_per_slice == int(case["metrics"]["cost"])  # > 2^64 on cfg2
    assert plan.width == case["metrics"]["width"]
    for ent in case["sliced"]:
        p2 = SlicedPlan(tn, tree, ent["labels"])
        assert p2.ops_per_slice * p2.d == int(ent["Cs"]) and p2.width == ent["Ws"]
        p2.close()
    plan.close()


def test_native_errors_mirror_reference():
    tn = gen.random_regular(10, 3, seed=1)
    from paper_2002_01935_b200.harness.paths import greedy_tree
    tree = greedy_tree(tn)
    with pytest.raises(ValueError):
        SlicedPlan(tn, tree, ["nope"])
    with pytest.raises(ValueError):
        SlicedPlan(tn, tree, ["e0", "e0"])
    bad = ContractionTree(tuple(range(1, 11)), tree.pairs)
    with pytest.raises(ValueError):
        SlicedPlan(tn, bad, ())
    tn_out = tn.replace(output=("e0",))
    with pytest.raises(ValueError):
        SlicedPlan(tn_out, tree, ["e0"])


def test_vertex_kinds_and_hoisting():
    tn = gen.grid_circuit(5, 5, 16, seed=3)
    from paper_2002_01935_b200.harness.paths import best_greedy_tree
    from paper_2002_01935_b200.slicing import greedy_slice
    tree = best_greedy_tree(tn, trials=2)
    m = metrics(tree, tn)
    ss = greedy_slice(tree, tn, m.width - 3, restarts=2)
    plan = SlicedPlan(tn, tree, ss)
    st = plan.stats()
    info = plan.vertex_info()
    assert len(info) == tn.num_nodes - 1
    assert st["num_hoisted"] == sum(v["hoisted"] for v in info) > 0
    assert sum(v["macs"] for v in info) == plan.ops_per_slice
    assert plan.width == sliced_metrics(tree, tn, ss.labels)[0]
    plan.close()


def test_accepts_reference_objects():
    """The executor plugs under the reference's own objects: hypertn
    TensorNetwork + a greedy_sample tree (drivers/greedy.py:144)."""
    from paper_2002_01935_b200 import refpkg
    tn = gen.random_regular(16, 3, seed=2)
    assert type(tn) is refpkg.network.TensorNetwork
    rt = refpkg.greedy_sample(tn, 1.0, 0.0, 0)
    assert type(rt) is refpkg.tree.ContractionTree
    plan = SlicedPlan(tn, rt, list(tn.index_table)[:2])
    assert plan.ops_per_slice * plan.d == sliced_metrics(rt, tn, list(tn.index_table)[:2])[1]
    assert plan.ops_per_slice * 1 <= refpkg.metrics(rt, tn).cost * 4
    plan.close()


def test_no_forked_reference_modules():
    """The package carries no copy of the reference's data model / tree layer."""
    import os
    import paper_2002_01935_b200 as pkg
    d = os.path.dirname(pkg.__file__)
    assert not os.path.exists(os.path.join(d, "network.py"))
    assert not os.path.exists(os.path.join(d, "tree.py"))
    from paper_2002_01935_b200 import refpkg
    assert refpkg.network.__file__.startswith(refpkg.REF_INSTALL) or \
        refpkg.network.__file__.startswith(refpkg.REF_SOURCE)


def test_auto_slice_fits_budget():
    from paper_2002_01935_b200.slicing import auto_slice
    from paper_2002_01935_b200.harness.paths import best_greedy_tree
    tn = gen.grid_circuit(5, 5, 16, seed=2)
    tree = best_greedy_tree(tn, trials=2)
    big, need_big = auto_slice(tree, tn, 1 << 40)
    assert big.labels == () or big.Ws == metrics(tree, tn).width
    small, need_small = auto_slice(tree, tn, 4 << 20)
    assert need_small <= 0.9 * (4 << 20) and small.Ws <= big.Ws
    assert small.Cs >= big.Cs


def test_allreduce_argument_checks():
    """tnx_allreduce error behaviour needs no device: empty list, duplicate
    plan and unbound plans are refused with ValueError (no CUDA call made)."""
    from paper_2002_01935_b200.executor import allreduce_plans
    tn = gen.random_regular(12, 3, seed=1)
    from paper_2002_01935_b200.harness.paths import greedy_tree
    tree = greedy_tree(tn, seed=0)
    a = SlicedPlan(tn, tree, ())
    b = SlicedPlan(tn, tree, ())
    try:
        with pytest.raises(ValueError):
            allreduce_plans([])
        with pytest.raises(ValueError, match="twice"):
            allreduce_plans([a, a])
        with pytest.raises(ValueError, match="not bound"):
            allreduce_plans([a, b])
    finally:
        a.close()
        b.close()


def _raw_desc(dims, leaves, pairs, out=(), sliced=()):
    """Plan descriptor straight through the C ABI (no Python wrapper checks)."""
    import ctypes as C
    flat = [l for lv in leaves for l in lv]
    keep = []  # keep the ctypes arrays alive with the struct

    def arr(t, xs):
        a = (t * max(1, len(xs)))(*xs)
        keep.append(a)
        return a
    d = nat.PlanDesc(len(dims), arr(C.c_int64, dims), len(leaves), arr(C.c_int32, [len(l) for l in leaves]),
                     arr(C.c_int32, flat), arr(C.c_int32, [c for p in pairs for c in p]),
                     len(out), arr(C.c_int32, out), len(sliced), arr(C.c_int32, sliced),
                     nat.PREC_3XTF32, 0, 0, 0, 0.0)
    return d, keep


def test_c_abi_status_codes():
    """tnx_plan_create / run / result error paths: invalid descriptors give
    TNX_ERR_INVALID with a message, calls out of order give TNX_ERR_STATE;
    nothing touches a GPU."""
    import ctypes as C
    lib = nat.load()
    h = C.c_void_p()
    # matrix chain a-b-c: x[a,b] y[b,c] z[c,a] -> scalar
    good_leaves = [[0, 1], [1, 2], [2, 0]]
    d, keep = _raw_desc([2, 3, 4], good_leaves, [(0, 1), (3, 2)])
    assert lib.tnx_plan_create(C.byref(d), C.byref(h)) == nat.TNX_OK
    assert lib.tnx_run_slices(h, 0, 1, None) == nat.TNX_ERR_STATE
    assert b"bind" in lib.tnx_last_error()
    out = (C.c_double * 2)()
    assert lib.tnx_partial_result(h, out, 1, None) == nat.TNX_ERR_STATE
    assert lib.tnx_plan_destroy(h) == nat.TNX_OK
    bad = [
        _raw_desc([2, 3, 4], good_leaves, [(0, 1), (0, 2)]),          # leaf consumed twice
        _raw_desc([2, 3, 4], good_leaves, [(0, 1), (4, 2)]),          # vertex not yet built
        _raw_desc([2, 3, 4], [[0, 1], [1, 7], [2, 0]], [(0, 1), (3, 2)]),  # label id out of range
        _raw_desc([2, 3, 4], good_leaves, [(0, 1), (3, 2)], out=(0,), sliced=(0,)),  # sliced output
        _raw_desc([2, 0, 4], good_leaves, [(0, 1), (3, 2)]),          # zero dimension
    ]
    for d, keep in bad:
        h = C.c_void_p()
        rc = lib.tnx_plan_create(C.byref(d), C.byref(h))
        assert rc in (nat.TNX_ERR_INVALID, nat.TNX_ERR_DATA), rc
        assert lib.tnx_last_error(), "error message expected"
        assert not h.value
    assert lib.tnx_plan_create(None, C.byref(h)) == nat.TNX_ERR_INVALID
