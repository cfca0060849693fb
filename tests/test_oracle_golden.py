"""Pin the CPU oracle against outputs of the real reference (tests/golden)."""
import pytest

import oracle
from conftest import arr_from_json, golden_cases
from _util import case_objects, rel_err

CASES = golden_cases()


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_keep_sets_and_costs(case):
    tn, tree = case_objects(case)
    terms = oracle.vertex_terms(tn, tree)
    assert [list(t) for t in terms] == case["keep_ordered"]
    W, C = oracle.width_cost(tn, tree)
    assert C == int(case["metrics"]["cost"])
    assert W == pytest.approx(case["metrics"]["width"], abs=0)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_values(case):
    tn, tree = case_objects(case)
    for ent in case["sliced"]:
        S = tuple(ent["labels"])
        Ws, Cper = oracle.width_cost(tn, tree, S)
        assert Ws == pytest.approx(ent["Ws"], abs=0)
        assert Cper * ent["d"] == int(ent["Cs"])
        if "value" not in ent:
            continue
        val, exp10, ops = oracle.contract_sliced(tn, tree, S)
        assert ops == int(ent["Cs"])
        ref = arr_from_json(ent["value"])
        assert rel_err(val, ref) <= 1e-12
        for sid, v in ent.get("per_slice", {}).items():
            got, _, _ = oracle.contract_sliced(tn, tree, S, slice_ids=[int(sid)])
            assert rel_err(got, arr_from_json(v)) <= 1e-12


def test_oracle_strip_exponent_invariant():
    case = [c for c in CASES if c["name"] == "cfg1_3reg50_greedy"][0]
    tn, tree = case_objects(case)
    v0, e0, _ = oracle.contract(tn, tree)
    v1, e1, _ = oracle.contract(tn, tree, strip_exponent=True)
    assert abs(v1 * 10.0 ** e1 - v0) <= 1e-12 * abs(v0)


def test_oracle_circuit_statevector():
    for case in CASES:
        if "statevector_amplitude" not in case:
            continue
        tn, tree = case_objects(case)
        val, _, _ = oracle.contract(tn, tree)
        sv = arr_from_json(case["statevector_amplitude"])
        assert abs(val - complex(sv)) <= 1e-12


def test_oracle_brute_force_random():
    from paper_2002_01935_b200.harness.generators import random_hyper_network
    from paper_2002_01935_b200.harness.paths import greedy_tree
    for seed in range(30):
        tn = random_hyper_network(6, 9, seed=seed)
        if tn.state_space() > 2 ** 16:
            continue
        tree = greedy_tree(tn, seed=seed)
        val, _, _ = oracle.contract(tn, tree)
        assert rel_err(val, oracle.brute_force(tn)) <= 1e-10


@pytest.mark.parametrize("rows,cols,depth", [(3, 4, 10), (4, 4, 12)])
def test_diagonal_reduced_circuit_amplitudes(rows, cols, depth):
    """Diagonal-reduced circuits (CZ / T as hyperedge nodes, hyperedge-safe
    rank simplification) give the statevector amplitude, like the split form."""
    import numpy as np
    from paper_2002_01935_b200.harness import generators as gen
    from paper_2002_01935_b200.harness.paths import greedy_tree
    for seed in range(2):
        bits = "".join(str(b) for b in np.random.default_rng(seed).integers(0, 2, rows * cols))
        ref = gen.circuit_statevector_amplitude(rows, cols, depth, seed=seed, bitstring=bits)
        for simplify in (False, True):
            tn = gen.grid_circuit(rows, cols, depth, seed=seed, bitstring=bits, simplify=simplify, diag=True)
            if not simplify:
                assert any(sum(l in nd.indices for nd in tn.nodes) > 2 for l in tn.index_table)
            val, _, _ = oracle.contract(tn, greedy_tree(tn))
            assert abs(val - ref) <= 1e-10 * max(1.0, abs(ref))
