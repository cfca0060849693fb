"""Contraction trees and their exact bookkeeping (keep sets, cost, width).

Drop-in mirror of the reference's tree layer for the hot path:

* ``ContractionTree(leaves, pairs)`` SSA form, validation, linear <-> SSA
  conversion -- `/root/reference/pkg/src/hypertn/tree.py:32-113`
* ``annotate_incidence(tree, tn)`` -- tree.py:137-169, using the label-count
  saturation algebra of ``HyperView`` (hypergraph.py:39-57, 90-131):
  a label stays live on a fragment while the number of leaves below it that
  carry the label is smaller than its total appearance count (carriers + 1
  if the label is an output).  The key order of each merged count dict is
  "survivors of a in a's order, then b's new labels in b's order"
  (hypergraph.py:106-119) -- this is also the natural output order of the
  reference's ``pairwise_contract`` (dense.py:74-75).
* ``metrics(tree, tn)`` -- tree.py:172-190 (W over internal vertices, exact
  integer C, flops = 8 C, n == 1 special case).
* path documents -- tree.py:195-223.

All integer quantities are Python ints (C exceeds 2^64 on the benchmark
trees).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

__all__ = ["PathMetrics", "ContractionTree", "LabelAlgebra", "Annotation",
           "annotate_incidence", "metrics", "tree_to_path_dict",
           "tree_from_path_dict"]


@dataclass(frozen=True)
class PathMetrics:
    """Width / cost summary (reference tree.py:15-29)."""
    width: float
    cost: int
    log10_cost: float
    flops: int
    peak_memory_elements: int


class ContractionTree:
    """Rooted binary tree in SSA pair form: leaf position i has id i (network
    node ``leaves[i]``), merge k creates id n + k (reference tree.py:32-57)."""

    __slots__ = ("leaves", "pairs", "_ann")

    def __init__(self, leaves, pairs):
        self.leaves = tuple(leaves)
        self.pairs = tuple((int(a), int(b)) for a, b in pairs)
        self._ann = None
        n = len(self.leaves)
        if len(set(self.leaves)) != n:
            raise ValueError("duplicate leaf ids")
        if n == 0:
            raise ValueError("empty tree")
        if len(self.pairs) != n - 1:
            raise ValueError(f"{len(self.pairs)} merge pairs for {n} leaves, need {n - 1}")
        used = set()
        for k, pair in enumerate(self.pairs):
            for c in pair:
                if c < 0 or c >= n + k:
                    raise ValueError(f"pair {k} references unbuilt vertex {c}")
                if c in used:
                    raise ValueError(f"vertex {c} consumed twice")
                used.add(c)

    @property
    def n(self):
        return len(self.leaves)

    @property
    def root(self):
        return 2 * self.n - 2 if self.n > 1 else 0

    def children(self, v):
        return self.pairs[v - self.n]

    def is_leaf(self, v):
        return v < self.n

    @property
    def incidence(self):
        """SSA vertex -> frozenset of labels (None until annotated)."""
        return None if self._ann is None else self._ann.label_sets()

    @classmethod
    def from_linear(cls, path, leaves):
        """Linear position-pair path -> tree (reference tree.py:81-98)."""
        n = len(leaves)
        live = list(range(n))
        pairs = []
        for step, (i, j) in enumerate(path):
            if i == j or not (0 <= i < len(live)) or not (0 <= j < len(live)):
                raise ValueError(f"step {step}: positions ({i}, {j}) invalid for "
                                 f"{len(live)} remaining tensors")
            a, b = live[i], live[j]
            for p in (max(i, j), min(i, j)):
                del live[p]
            live.append(n + step)
            pairs.append((a, b))
        return cls(leaves, pairs)

    def to_linear(self):
        """Inverse of :meth:`from_linear` (reference tree.py:100-113)."""
        live = list(range(self.n))
        path = []
        for k, (a, b) in enumerate(self.pairs):
            i, j = sorted((live.index(a), live.index(b)))
            path.append((i, j))
            del live[j]
            del live[i]
            live.append(self.n + k)
        return path


class LabelAlgebra:
    """Interned label-count algebra over a network (hypergraph.py:12-131).

    ``labels`` are interned in ``tn.index_table`` insertion order; a leaf's
    count dict lists its labels in ``node.indices`` order with count 1.
    """

    __slots__ = ("labels", "label_ids", "dims", "appearances", "leaf_terms",
                 "item_ids")

    def __init__(self, tn):
        self.labels = list(tn.index_table)
        self.label_ids = {lbl: i for i, lbl in enumerate(self.labels)}
        self.dims = [tn.index_table[lbl] for lbl in self.labels]
        app = [0] * len(self.labels)
        terms, ids = [], []
        for nd in tn.nodes:
            term = {}
            for lbl in nd.indices:
                li = self.label_ids[lbl]
                term[li] = 1
                app[li] += 1
            terms.append(term)
            ids.append(nd.id)
        for lbl in tn.output:
            app[self.label_ids[lbl]] += 1
        self.appearances = app
        self.leaf_terms = terms
        self.item_ids = ids

    def merge(self, a, b):
        """Sum counts; drop saturated labels.  Order: a's survivors, then b's
        new labels (hypergraph.py:106-119)."""
        app = self.appearances
        out = {}
        for li, ca in a.items():
            c = ca + b.get(li, 0)
            if c < app[li]:
                out[li] = c
        for li, cb in b.items():
            if li not in a and cb < app[li]:
                out[li] = cb
        return out

    def union_product(self, a, b):
        """Exact MAC count of merging a and b (hypergraph.py:121-131)."""
        dims = self.dims
        p = 1
        for li in a:
            p *= dims[li]
        for li in b:
            if li not in a:
                p *= dims[li]
        return p

    def size(self, term):
        dims = self.dims
        p = 1
        for li in term:
            p *= dims[li]
        return p


class Annotation:
    """Incidence sets and congestion numbers of one (tree, network) pair
    (reference ``TreeAnnotation``, tree.py:116-134)."""

    __slots__ = ("tn", "algebra", "terms", "cost_terms", "result_sizes")

    def __init__(self, tn, algebra, terms, cost_terms, result_sizes):
        self.tn = tn
        self.algebra = algebra
        self.terms = terms            # ssa vertex -> ordered {label_id: count}
        self.cost_terms = cost_terms  # internal vertex -> union product
        self.result_sizes = result_sizes

    # reference spelling of the two attributes kept for drop-in use
    @property
    def view(self):
        return self.algebra

    @property
    def counts(self):
        return self.terms

    def label_sets(self):
        names = self.algebra.labels
        return {v: frozenset(names[li] for li in t) for v, t in enumerate(self.terms)}

    def ordered_labels(self, v):
        """Labels of vertex v in the reference's natural order."""
        names = self.algebra.labels
        return tuple(names[li] for li in self.terms[v])

    def set_ids(self, v):
        return self.terms[v].keys()


def annotate_incidence(tree, tn):
    """Attach every incidence set of ``tree`` over ``tn`` (tree.py:137-169).

    Cached on the tree while it is annotated against the same network object.
    """
    if tree._ann is not None and tree._ann.tn is tn:
        return tree
    alg = LabelAlgebra(tn)
    if sorted(tree.leaves) != sorted(alg.item_ids):
        raise ValueError("tree leaves do not match network node ids")
    where = {nid: p for p, nid in enumerate(alg.item_ids)}
    n = tree.n
    terms = [None] * (2 * n - 1 if n > 1 else 1)
    for i, nid in enumerate(tree.leaves):
        terms[i] = alg.leaf_terms[where[nid]]
    cost_terms, sizes = {}, {}
    for k, (a, b) in enumerate(tree.pairs):
        v = n + k
        cost_terms[v] = alg.union_product(terms[a], terms[b])
        terms[v] = alg.merge(terms[a], terms[b])
        sizes[v] = alg.size(terms[v])
    tree._ann = Annotation(tn, alg, terms, cost_terms, sizes)
    return tree


def metrics(tree, tn):
    """W, C, log10 C, flops = 8 C, peak (reference tree.py:172-190)."""
    annotate_incidence(tree, tn)
    ann = tree._ann
    if tree.n == 1:
        out_size = 1
        for lbl in tn.output:
            out_size *= tn.index_table[lbl]
        return PathMetrics(math.log2(out_size), 0, float("-inf"), 0, out_size)
    cost = sum(ann.cost_terms.values())
    peak = max(ann.result_sizes.values())
    return PathMetrics(math.log2(peak) if peak > 0 else 0.0, cost,
                       math.log10(cost) if cost > 0 else float("-inf"),
                       8 * cost, peak)


def tree_to_path_dict(tree, fmt="linear"):
    """Path document (tree.py:195-208)."""
    if fmt == "linear":
        return {"format": "linear", "path": [list(p) for p in tree.to_linear()]}
    if fmt == "ssa":
        return {"format": "ssa", "num_leaves": tree.n,
                "path": [list(p) for p in tree.pairs]}
    raise ValueError(f"unknown path format {fmt!r}")


def tree_from_path_dict(obj, tn):
    """Load a path document against a network, leaves in node order
    (tree.py:211-223)."""
    if not isinstance(obj, dict) or "format" not in obj or "path" not in obj:
        raise ValueError("path document needs 'format' and 'path'")
    leaves = tn.node_ids
    fmt = obj["format"]
    if fmt == "linear":
        return ContractionTree.from_linear([tuple(p) for p in obj["path"]], leaves)
    if fmt == "ssa":
        if obj.get("num_leaves", len(leaves)) != len(leaves):
            raise ValueError("ssa path leaf count does not match network")
        return ContractionTree(leaves, [tuple(p) for p in obj["path"]])
    raise ValueError(f"unknown path format {fmt!r}")
