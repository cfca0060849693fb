"""Benchmark workloads: BASELINE.json configs as (network, tree, slice set).

Networks are regenerated deterministically (``generators``); trees are the
ones the REFERENCE drivers produced in the build container
(``benchdata/<name>.tree.json`` written by ``benchdata/make_trees.py``); the
slice set comes from this package's ``greedy_slice`` (the
reference ships no slicer).  Harness code, not product.
"""

from __future__ import annotations

import json
import os

from . import generators as gen
from .paths import best_greedy_tree
from ..slicing import greedy_slice, SliceSet
from ..refpkg import ContractionTree, metrics

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
BENCHDATA = os.path.join(REPO, "benchdata")

CONFIGS = {
    "cfg1_3reg50": dict(make=lambda: gen.random_regular(50, 3, seed=0), ws=None,
                        desc="random 3-regular network, 50 tensors, bond dim 2"),
    "cfg2_5reg100": dict(make=lambda: gen.random_regular(100, 5, seed=0), ws=28,
                         desc="random 5-regular network, 100 tensors, bond dim 2"),
    "cfg3_lattice20": dict(make=lambda: gen.square_lattice(20, seed=0), ws=None,
                           desc="20x20 OBC square lattice, bond dim 2, scalar"),
    "cfg3g_lattice20": dict(make=lambda: gen.square_lattice(20, seed=0), ws=None,
                            desc="20x20 OBC square lattice, bond dim 2, scalar; plain greedy tree"),
    "cfg4_7x7_d40": dict(make=lambda: gen.grid_circuit(7, 7, 40, seed=0), ws=27,
                         desc="rectangular 7x7 (1+40+1) random circuit amplitude, 742 rank-3 tensors"),
    "cfg4g_7x7_d40": dict(make=lambda: gen.grid_circuit(7, 7, 40, seed=0), ws=27,
                          desc="7x7 (1+40+1) circuit amplitude, greedy-driver tree (round-1 bench tree)"),
    # parity-only companions of cfg4 (same generator, shallower): the full
    # amplitude is computable by the CPU oracle
    "cfg4p_7x7_d16": dict(make=lambda: gen.grid_circuit(7, 7, 16, seed=0), ws=16,
                          desc="7x7 (1+16+1) circuit amplitude (parity companion of cfg4)"),
    "cfg4p_7x7_d20": dict(make=lambda: gen.grid_circuit(7, 7, 20, seed=0), ws=21,
                          desc="7x7 (1+20+1) circuit amplitude (parity companion of cfg4)"),
    "cfg4p_7x7_d24": dict(make=lambda: gen.grid_circuit(7, 7, 24, seed=0), ws=27,
                          desc="7x7 (1+24+1) circuit amplitude (parity companion of cfg4; oracle sliced at W_s=27)"),
    "cfg5_syc53_m12": dict(make=lambda: gen.sycamore_circuit(12, seed=0), ws=27,
                           desc="Sycamore-like 53-qubit m=12 circuit amplitude, synthetic fSim"),
    # the cfg4 circuit diagonal-reduced (CZ and T gates as hyperedge nodes,
    # SPEC.md:241-248): hyperedge-heavy networks (batched GEMM / SIMT paths)
    "cfg4d_7x7_d40_diag": dict(make=lambda: gen.grid_circuit(7, 7, 40, seed=0, diag=True), ws=27,
                               desc="7x7 (1+40+1) circuit amplitude, diagonal-reduced (hyperedges)"),
    "cfg4dp_7x7_d20_diag": dict(make=lambda: gen.grid_circuit(7, 7, 20, seed=0, diag=True), ws=None,
                                desc="7x7 (1+20+1) diagonal-reduced amplitude (parity: equals cfg4p_7x7_d20)"),
}


def load_tree(name, tn):
    path = os.path.join(BENCHDATA, f"{name}.tree.json")
    if os.path.exists(path):
        with open(path) as fh:
            rec = json.load(fh)
        return ContractionTree(rec["tree"]["leaves"], [tuple(p) for p in rec["tree"]["pairs"]]), rec
    tree = best_greedy_tree(tn, trials=8)
    return tree, {"driver": "harness best_greedy_tree (no reference tree file)"}


def load_workload(name, ws=None, restarts=2, seed=0):
    cfg = CONFIGS[name]
    tn = cfg["make"]()
    tree, rec = load_tree(name, tn)
    ws = cfg["ws"] if ws is None else ws
    m = metrics(tree, tn)
    if ws is None or ws >= m.width:
        ss = SliceSet.from_labels(tree, tn, ())
    else:
        ss = greedy_slice(tree, tn, ws, restarts=restarts, seed=seed)
    return tn, tree, ss, {"tree_source": rec.get("driver"), "W": m.width,
                          "log10_C": m.log10_cost, "desc": cfg["desc"]}
