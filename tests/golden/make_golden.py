"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``hypertn`` from ``/root/reference/pkg/src`` (read-only, never
copied) and records, for seeded networks and trees:

* keep sets in the reference's natural order (``annotate_incidence`` counts,
  tree.py:137-169 / hypergraph.py:106-119),
* ``metrics`` (tree.py:172-190): W, C, flops, peak, and per-vertex cost terms,
* sliced W_s / C_s by the SPEC formula evaluated on the
  reference's incidence sets,
* contraction values obtained by composing the reference's own numeric ops:
  ``fix_index`` (dense.py:161) on sliced leaves, ``pairwise_contract``
  (dense.py:61) per SSA pair with keep = incidence - S, ``transpose_to``
  (dense.py:36) at the root, summed over every slice assignment (the
  SPEC.md:524 loop -- the reference ships no executor),
* trees produced by the reference drivers (``greedy_sample``,
  ``optimal_dp``).

The JSON files written next to this script are committed; tests read only
those files (``/root/reference`` does not exist on the GPU box).
"""

from __future__ import annotations

import itertools
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from hypertn import network as rnet  # noqa: E402
from hypertn import tree as rtree  # noqa: E402
from hypertn import dense as rdense  # noqa: E402
from hypertn.drivers import greedy as rgreedy  # noqa: E402
from hypertn.drivers import optimal as roptimal  # noqa: E402

from paper_2002_01935_b200.harness import generators as gen  # noqa: E402


def to_ref(tn):
    """Our generator's network -> reference TensorNetwork (same content)."""
    nodes = [rnet.TensorNode(nd.id, nd.indices, nd.data) for nd in tn.nodes]
    return rnet.TensorNetwork(nodes, dict(tn.index_table), tn.output, tn.norm_exponent)


def ref_contract_slice(tn, tree, S, assign):
    rtree.annotate_incidence(tree, tn)
    inc = tree.incidence
    n = tree.n
    bufs = {}
    for i, nid in enumerate(tree.leaves):
        nd = tn.node(nid)
        t = rdense.DenseTensor(nd.indices, nd.data)
        for lbl in S:
            if lbl in t.labels:
                t = rdense.fix_index(t, lbl, assign[lbl])
        bufs[i] = t
    for k, (a, b) in enumerate(tree.pairs):
        v = n + k
        keep = set(inc[v]) - set(S)
        bufs[v] = rdense.pairwise_contract(bufs.pop(a), bufs.pop(b), keep)
    root = bufs[tree.root]
    extra = [l for l in root.labels if l not in tn.output]
    if extra:  # single-leaf tree: nested-sum definition sums non-output labels
        arr = root.array.sum(axis=tuple(root.labels.index(l) for l in extra))
        root = rdense.DenseTensor([l for l in root.labels if l not in extra], arr)
    return root.transpose_to(tn.output).array


def ref_contract_sliced(tn, tree, S, ids=None):
    dims = [tn.index_table[l] for l in S]
    combos = list(itertools.product(*[range(w) for w in dims]))
    if ids is not None:
        combos = [combos[i] for i in ids]
    total = None
    for c in combos:
        r = ref_contract_slice(tn, tree, S, dict(zip(S, c)))
        total = r if total is None else total + r
    return total


def ref_sliced_metrics(tn, tree, S):
    rtree.annotate_incidence(tree, tn)
    inc = tree.incidence
    n = tree.n
    dims = tn.index_table
    d = 1
    for l in S:
        d *= dims[l]
    if n == 1:
        return rtree.metrics(tree, tn).width, 0, d
    per, peak = 0, 0
    for k, (a, b) in enumerate(tree.pairs):
        v = n + k
        u = (inc[a] | inc[b]) - set(S)
        p = 1
        for l in u:
            p *= dims[l]
        per += p
        q = 1
        for l in inc[v] - set(S):
            q *= dims[l]
        peak = max(peak, q)
    return math.log2(peak), d * per, d


def arr_json(a):
    a = np.asarray(a, dtype=np.complex128)
    return {"shape": list(a.shape), "re": a.real.ravel().tolist(), "im": a.imag.ravel().tolist()}


def case_record(name, tn, tree, slice_sets, per_slice_ids=(0,)):
    rtree.annotate_incidence(tree, tn)
    ann = tree._ann
    names = ann.view.labels
    m = rtree.metrics(tree, tn)
    rec = {
        "name": name,
        "network": rnet.network_to_dict(tn),
        "tree": {"leaves": list(tree.leaves), "pairs": [list(p) for p in tree.pairs]},
        "keep_ordered": [[names[li] for li in c] for c in ann.counts],
        "cost_terms": {str(v): str(c) for v, c in ann.cost_terms.items()},
        "metrics": {"width": m.width, "cost": str(m.cost), "flops": str(m.flops),
                    "peak": str(m.peak_memory_elements)},
        "sliced": [],
    }
    for S in slice_sets:
        ws, cs, d = ref_sliced_metrics(tn, tree, S)
        ent = {"labels": list(S), "Ws": ws, "Cs": str(cs), "d": d}
        if tn.has_all_data():
            ent["value"] = arr_json(ref_contract_sliced(tn, tree, S))
            ent["per_slice"] = {str(i): arr_json(ref_contract_sliced(tn, tree, S, [i]))
                                for i in per_slice_ids if i < d}
        rec["sliced"].append(ent)
    return rec


def kat_cases():
    out = []
    # SPEC.md:105-108 annotate_incidence KATs
    I2 = np.eye(2)
    tn = to_ref(gen.TensorNetwork([gen.TensorNode(0, "ab", np.arange(4).reshape(2, 2) + 1.0),
                                   gen.TensorNode(1, "bc", np.arange(4).reshape(2, 2) - 1.5j)],
                                  {"a": 2, "b": 2, "c": 2}, ("a", "c")))
    out.append(case_record("kat_ab_bc_ac", tn, rtree.ContractionTree((0, 1), [(0, 1)]), [()]))
    tn = to_ref(rnet.from_arrays("a,a,a->", [np.array([1.0, 2.0]), np.array([3.0, -1.0]),
                                             np.array([0.5, 0.25j])]))
    out.append(case_record("kat_hyper_aaa", tn, rtree.ContractionTree((0, 1, 2), [(1, 2), (0, 3)]), [()]))
    tn = to_ref(rnet.from_arrays("ab,ab->", [np.arange(6).reshape(2, 3) + 0.5, np.ones((2, 3)) * 1j]))
    out.append(case_record("kat_closed_pair", tn, rtree.ContractionTree((0, 1), [(0, 1)]), [()]))
    # SPEC.md:114-117 matrix chain (2x4)(4x8)(8x2)
    rng = np.random.default_rng(3)
    arrs = [rng.standard_normal((2, 4)), rng.standard_normal((4, 8)), rng.standard_normal((8, 2))]
    tn = to_ref(rnet.from_arrays("ab,bc,cd->ad", arrs))
    out.append(case_record("kat_chain_ABC", tn, rtree.ContractionTree((0, 1, 2), [(0, 1), (3, 2)]),
                           [(), ("c",)], per_slice_ids=(0, 7)))
    tn2 = to_ref(rnet.from_arrays("ab,bc,cd->", arrs))  # closed? no: a,d dangling summed
    out.append(case_record("kat_chain_opt", tn, roptimal.optimal_dp(tn), [()]))
    out.append(case_record("kat_chain_dangling", tn2, rtree.ContractionTree((0, 1, 2), [(0, 1), (3, 2)]),
                           [(), ("b",)]))
    # SPEC.md:181-184 I2 . I2 over "ab,ba->" = 2
    tn = to_ref(rnet.from_arrays("ab,ba->", [I2, I2]))
    out.append(case_record("kat_trace_identity", tn, rtree.ContractionTree((0, 1), [(0, 1)]), [(), ("a",)]))
    # Hadamard "ab,ab->ab"
    tn = to_ref(rnet.from_arrays("ab,ab->ab", [np.arange(4).reshape(2, 2) + 1.0, np.arange(4).reshape(2, 2) * 1j]))
    out.append(case_record("kat_hadamard", tn, rtree.ContractionTree((0, 1), [(0, 1)]), [()]))
    # single node network
    tn = to_ref(rnet.from_arrays("abc->ca", [np.arange(8).reshape(2, 2, 2) + 0.5j]))
    out.append(case_record("kat_single_node", tn, rtree.ContractionTree((0,), []), [()]))
    return out


def random_cases(count=40):
    out = []
    for seed in range(count):
        rng = np.random.default_rng(1000 + seed)
        nn = int(rng.integers(2, 10))
        nl = int(rng.integers(nn, 2 * nn + 3))
        tn = to_ref(gen.random_hyper_network(nn, nl, seed=seed, max_rank=5))
        if tn.state_space() > 2 ** 18:
            continue
        trees = [("greedy", rgreedy.greedy_sample(tn, alpha=float(rng.uniform(0, 2)),
                                                   tau=float(rng.choice([0.0, 0.5])), seed=seed))]
        if nn <= 8:
            trees.append(("optimal", roptimal.optimal_dp(tn)))
        closed = [l for l in tn.index_table if l not in tn.output and tn.carriers(l)]
        for tname, tree in trees:
            sets = [()]
            if closed:
                k = int(rng.integers(1, min(3, len(closed)) + 1))
                pick = rng.choice(len(closed), size=k, replace=False)
                sets.append(tuple(closed[int(i)] for i in pick))
            out.append(case_record(f"rand{seed}_{tname}", tn, tree, sets, per_slice_ids=(0, 1)))
    return out


def config_cases():
    out = []
    # configs[0]: random 3-regular n=50, reference greedy tree (alpha=1, tau=0, seed=0)
    tn = to_ref(gen.random_regular(50, 3, seed=0))
    tree = rgreedy.greedy_sample(tn, 1.0, 0.0, 0)
    rec = case_record("cfg1_3reg50_greedy", tn, tree, [()])
    labels = [l for l in tn.index_table][:3]
    ws, cs, d = ref_sliced_metrics(tn, tree, labels)
    rec["sliced"].append({"labels": labels, "Ws": ws, "Cs": str(cs), "d": d,
                          "value": arr_json(ref_contract_sliced(tn, tree, labels)),
                          "per_slice": {str(i): arr_json(ref_contract_sliced(tn, tree, labels, [i]))
                                        for i in (0, 5)}})
    out.append(rec)
    # small circuits: 3x3 depth 8 and 4x4 depth 10, reference greedy tree
    for (r, c, dep, seed) in ((3, 3, 8, 1), (4, 4, 10, 2)):
        tn = to_ref(gen.grid_circuit(r, c, dep, seed=seed))
        tree = rgreedy.greedy_sample(tn, 1.0, 0.0, seed)
        rec = case_record(f"circuit_{r}x{c}_d{dep}", tn, tree, [()])
        rec["statevector_amplitude"] = arr_json(gen.circuit_statevector_amplitude(r, c, dep, seed=seed))
        out.append(rec)
    return out


def structural_cases():
    """Bookkeeping-only goldens for the big configurations (no values)."""
    out = []
    for name, tn, seed in (("cfg2_5reg100", gen.random_regular(100, 5, seed=0), 0),
                           ("cfg3_lattice20", gen.square_lattice(20, seed=0), 0),
                           ("cfg4_7x7_d40", gen.grid_circuit(7, 7, 40, seed=0), 0)):
        rtn = to_ref(tn)
        tree = rgreedy.greedy_sample(rtn, 1.0, 0.0, seed)
        rtree.annotate_incidence(tree, rtn)
        m = rtree.metrics(tree, rtn)
        names = tree._ann.view.labels
        labels = list(rtn.index_table)[: 12]
        ws, cs, d = ref_sliced_metrics(rtn, tree, labels)
        out.append({"name": name, "tree": {"leaves": list(tree.leaves),
                                             "pairs": [list(p) for p in tree.pairs]},
                    "keep_ordered": [[names[li] for li in cnt] for cnt in tree._ann.counts],
                    "metrics": {"width": m.width, "cost": str(m.cost), "flops": str(m.flops),
                                "peak": str(m.peak_memory_elements)},
                    "sliced": [{"labels": labels, "Ws": ws, "Cs": str(cs), "d": d}]})
    return out


def main():
    data = {"kat": kat_cases(), "random": random_cases(), "configs": config_cases()}
    with open(os.path.join(HERE, "reference_cases.json"), "w") as fh:
        json.dump(data, fh)
    with open(os.path.join(HERE, "reference_structural.json"), "w") as fh:
        json.dump(structural_cases(), fh)
    print("cases:", {k: len(v) for k, v in data.items()})


if __name__ == "__main__":
    main()
