"""Bit-exact host bookkeeping vs the reference (tests/golden)."""
import itertools
import math

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from _util import case_objects
from paper_2002_01935_b200.refpkg import network_from_dict, network_to_dict, DataError, from_arrays
from paper_2002_01935_b200.refpkg import (ContractionTree, annotate_incidence, metrics,
                                        tree_to_path_dict, tree_from_path_dict, ordered_labels)
from paper_2002_01935_b200.slicing import (SliceSet, sliced_metrics, greedy_slice,
                                           slice_digits, slice_assignment, iter_slice_assignments)
from paper_2002_01935_b200.harness import generators as gen

CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_annotate_and_metrics(case):
    tn, tree = case_objects(case)
    annotate_incidence(tree, tn)
    order = [list(ordered_labels(tree, tn, v)) for v in range(len(tree._ann.counts))]
    assert order == case["keep_ordered"]
    m = metrics(tree, tn)
    assert m.cost == int(case["metrics"]["cost"])
    assert m.flops == int(case["metrics"]["flops"])
    assert m.peak_memory_elements == int(case["metrics"]["peak"])
    assert m.width == case["metrics"]["width"]
    assert {str(k): str(v) for k, v in tree._ann.cost_terms.items()} == case["cost_terms"]
    for ent in case["sliced"]:
        ws, cs = sliced_metrics(tree, tn, ent["labels"])
        assert ws == ent["Ws"] and cs == int(ent["Cs"])
        assert SliceSet.from_labels(tree, tn, ent["labels"]).d == ent["d"]


STRUCT = load_golden("reference_structural.json")


@pytest.mark.parametrize("case", STRUCT, ids=[c["name"] for c in STRUCT])
def test_structural_configs(case):
    name = case["name"]
    tn = {"cfg2_5reg100": lambda: gen.random_regular(100, 5, seed=0),
          "cfg3_lattice20": lambda: gen.square_lattice(20, seed=0),
          "cfg4_7x7_d40": lambda: gen.grid_circuit(7, 7, 40, seed=0)}[name]()
    tree = ContractionTree(case["tree"]["leaves"], [tuple(p) for p in case["tree"]["pairs"]])
    annotate_incidence(tree, tn)
    assert [list(ordered_labels(tree, tn, v)) for v in range(2 * tree.n - 1)] == case["keep_ordered"]
    m = metrics(tree, tn)
    assert m.cost == int(case["metrics"]["cost"]) and m.width == case["metrics"]["width"]
    for ent in case["sliced"]:
        ws, cs = sliced_metrics(tree, tn, ent["labels"])
        assert ws == ent["Ws"] and cs == int(ent["Cs"])


def test_spec_kat_matrix_chain():
    rng = np.random.default_rng(0)
    tn = from_arrays("ab,bc,cd->ad", [rng.standard_normal((2, 4)), rng.standard_normal((4, 8)),
                                      rng.standard_normal((8, 2))])
    t1 = ContractionTree((0, 1, 2), [(0, 1), (3, 2)])
    m = metrics(t1, tn)
    assert (m.cost, m.width, m.flops) == (96, 4.0, 768)
    t2 = ContractionTree((0, 1, 2), [(1, 2), (0, 3)])
    m = metrics(t2, tn)
    assert (m.cost, m.width) == (80, 3.0)
    # slicing c on ((AB)C): per-slice C = 12, C_s = 96
    ws, cs = sliced_metrics(t1, tn, ["c"])
    assert cs == 96
    ss = SliceSet.from_labels(t1, tn, ["c"])
    assert ss.per_slice_cost == 12 and ss.d == 8
    assert sliced_metrics(t1, tn, []) == (4.0, 96)
    with pytest.raises(ValueError):
        sliced_metrics(t1, tn, ["a"])  # output label


def test_tree_validation_errors():
    with pytest.raises(ValueError):
        ContractionTree((0, 1, 2), [(0, 1)])
    with pytest.raises(ValueError):
        ContractionTree((0, 1, 2), [(0, 1), (0, 3)])
    with pytest.raises(ValueError):
        ContractionTree((0, 1, 2), [(0, 5), (1, 2)])
    with pytest.raises(ValueError):
        ContractionTree((0, 0), [(0, 1)])


def test_linear_ssa_roundtrip():
    tn = gen.random_regular(12, 3, seed=4)
    from paper_2002_01935_b200.harness.paths import greedy_tree
    tree = greedy_tree(tn, seed=1)
    lin = tree.to_linear()
    t2 = ContractionTree.from_linear(lin, tree.leaves)
    assert t2.pairs == tree.pairs
    for fmt in ("linear", "ssa"):
        t3 = tree_from_path_dict(tree_to_path_dict(tree, fmt), tn)
        assert metrics(t3, tn).cost == metrics(tree, tn).cost
    with pytest.raises(ValueError):
        ContractionTree.from_linear([(0, 5)], (0, 1, 2))


def test_json_roundtrip_bit_exact():
    tn = gen.random_hyper_network(7, 10, seed=3)
    tn2 = network_from_dict(network_to_dict(tn))
    for a, b in zip(tn.nodes, tn2.nodes):
        assert a.indices == b.indices and np.array_equal(a.data, b.data)
    assert tn2.output == tn.output and tn2.index_table == tn.index_table
    bad = network_to_dict(tn)
    bad["tensors"][0]["data"] = "!!!"
    with pytest.raises(DataError):
        network_from_dict(bad)


def test_slice_enumeration_bit_exact():
    dims = [2, 3, 1, 2, 4]
    combos = list(itertools.product(*[range(w) for w in dims]))
    d = math.prod(dims)
    for s in range(d):
        assert slice_digits(dims, s) == combos[s]
        assert slice_digits(dims, s) == tuple(int(x) for x in np.unravel_index(s, dims))
    with pytest.raises(ValueError):
        slice_digits(dims, d)
    big = [2] * 40
    s = (1 << 39) + 12345
    dg = slice_digits(big, s)
    assert int("".join(map(str, dg)), 2) == s


def test_greedy_slice_invariants():
    tn = gen.square_lattice(6, seed=0)
    from paper_2002_01935_b200.harness.paths import best_greedy_tree
    tree = best_greedy_tree(tn, trials=4)
    m = metrics(tree, tn)
    for target in (m.width, m.width - 1, m.width - 3):
        ss = greedy_slice(tree, tn, target, restarts=4, seed=1)
        assert ss.Ws <= target
        assert m.cost <= ss.Cs <= ss.d * m.cost
        if target >= m.width:
            assert ss.labels == ()
    a = greedy_slice(tree, tn, m.width - 2, restarts=3, seed=7)
    b = greedy_slice(tree, tn, m.width - 2, restarts=3, seed=7)
    assert a.labels == b.labels
    with pytest.raises(ValueError):
        greedy_slice(tree, tn, 1.0)
    # monotonicity: adding labels never increases W_s
    prev = m.width
    for k in range(1, len(a.labels) + 1):
        ws, _ = sliced_metrics(tree, tn, a.labels[:k])
        assert ws <= prev
        prev = ws
    asg = list(iter_slice_assignments(tn, a))
    assert len(asg) == a.d and asg[3] == slice_assignment(tn, a, 3)


def test_amplitude_projection_open_markers():
    """_project fixes digits and keeps 'x' / '*' positions as outputs in qubit
    order (host logic only)."""
    import numpy as np
    from paper_2002_01935_b200.executor import _project
    from paper_2002_01935_b200.refpkg import TensorNetwork, TensorNode
    rng = np.random.default_rng(0)
    a = rng.standard_normal((2, 2, 3)) + 0j
    b = rng.standard_normal((2, 3)) + 0j
    tn = TensorNetwork([TensorNode(0, ["q0", "q1", "k"], a), TensorNode(1, ["q2", "k"], b)],
                       {"q0": 2, "q1": 2, "q2": 2, "k": 3}, ("q0", "q1", "q2"))
    p = _project(tn, "x1*")
    assert p.output == ("q0", "q2")
    assert p.node(0).indices == ("q0", "k") and p.node(1).indices == ("q2", "k")
    assert np.array_equal(p.node(0).data, a[:, 1, :])
    assert "q1" not in p.index_table
    with pytest.raises(ValueError):
        _project(tn, "x1")
    with pytest.raises(ValueError):
        _project(tn, "a10")


def test_slice_runs_and_device_shares():
    from paper_2002_01935_b200.executor import _slice_runs, _split_runs
    assert _slice_runs(16, None) == [(0, 16)]
    assert _slice_runs(16, range(3, 9)) == [(3, 9)]
    assert _slice_runs(16, [0, 7]) == [(0, 1), (7, 8)]
    assert _slice_runs(16, [4, 5, 6, 1, 2]) == [(4, 7), (1, 3)]
    with pytest.raises(ValueError):
        _slice_runs(16, [16])
    with pytest.raises(ValueError):
        _slice_runs(16, range(0, 8, 2))
    runs = [(0, 5), (10, 13)]
    for G in (1, 2, 3, 8):
        shares = _split_runs(runs, G)
        flat = [s for sh in shares for a, b in sh for s in range(a, b)]
        assert flat == list(range(0, 5)) + list(range(10, 13))
        sizes = [sum(b - a for a, b in sh) for sh in shares]
        assert max(sizes) - min(sizes) <= 1
