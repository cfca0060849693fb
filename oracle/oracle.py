"""CPU ORACLE for the sliced contraction-tree executor -- TEST INFRASTRUCTURE.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The B200 product path
(``paper_2002_01935_b200``) never imports or calls anything here.

The reference ships the per-op building blocks but not the executor loop
(`/root/reference/SPEC.md:510-558`, ``contract`` / ``contract_sliced`` are
spec-only).  This oracle is that loop, written over the REFERENCE'S OWN
functions, called directly from the installed ``hypertn`` (``baseline/_ref``,
located by ``paper_2002_01935_b200.refpkg``):

* keep sets   -- ``hypertn.tree.annotate_incidence`` (`tree.py:137-169`), i.e.
  the saturation rule of ``HyperView.merge_counts`` (`hypergraph.py:106-119`);
* per-pair op -- ``hypertn.dense.pairwise_contract`` (`dense.py:61-76`, which
  evaluates ``np.einsum(..., optimize=True)``, `dense.py:47-58`).  Only a pair
  whose label union exceeds the reference's 52-symbol limit (`dense.py:10`,
  `:49-52`) -- which the reference itself cannot contract -- goes through the
  restated batch/M/N/K matmul ``_matmul_pair`` below;
* op count    -- the union product (`hypergraph.py:121-131`) per vertex;
* slicing     -- ``hypertn.dense.fix_index`` (`dense.py:161-170`) on every
  leaf carrying a sliced label; slice ids enumerate mixed-radix, last label
  fastest;
* root        -- ``DenseTensor.transpose_to(tn.output)`` (`dense.py:36-41`);
* reduction   -- compensated (Kahan) complex128 summation over slices
  (SPEC.md:551); ``strip_exponent`` renormalisation.

Parity pinning: ``tests/golden/make_golden.py`` records outputs of the
reference functions on seeded networks as ``tests/golden/*.json``;
``tests/test_oracle_golden.py`` checks this oracle against them.
"""

from __future__ import annotations

import math
import string

import numpy as np

from paper_2002_01935_b200.refpkg import dense as _rd, annotate_incidence as _annotate

_LETTERS = string.ascii_letters  # dense.py:10 -- at most 52 labels per pair


# ------------------------------------------------------------ bookkeeping
def appearances(tn):
    """label -> (#carrier leaves + 1 if output) (hypergraph.py:50-56)."""
    app = {lbl: 0 for lbl in tn.index_table}
    for nd in tn.nodes:
        for lbl in nd.indices:
            app[lbl] += 1
    for lbl in tn.output:
        app[lbl] += 1
    return app


def vertex_terms(tn, tree):
    """Ordered {label: count} per SSA vertex, from the reference's
    ``annotate_incidence`` (tree.py:137-169)."""
    _annotate(tree, tn)
    names = tree._ann.view.labels
    return [{names[li]: c for li, c in cnt.items()} for cnt in tree._ann.counts]


def cost_terms(tn, tree, sliced=()):
    """Per-vertex MAC counts with ``sliced`` removed (exact ints)."""
    terms = vertex_terms(tn, tree)
    dims = tn.index_table
    S = set(sliced)
    out = []
    for a, b in tree.pairs:
        u = (set(terms[a]) | set(terms[b])) - S
        p = 1
        for lbl in u:
            p *= dims[lbl]
        out.append(p)
    return out


def width_cost(tn, tree, sliced=()):
    """(W, C) -- or (W_s, per-slice C) with ``sliced`` removed."""
    terms = vertex_terms(tn, tree)
    n = len(tree.leaves)
    if n == 1:
        size = 1
        for lbl in tn.output:
            size *= tn.index_table[lbl]
        return math.log2(size), 0
    S = set(sliced)
    peak = 0
    for t in terms[n:]:
        p = 1
        for lbl in t:
            if lbl not in S:
                p *= tn.index_table[lbl]
        peak = max(peak, p)
    return math.log2(peak), sum(cost_terms(tn, tree, sliced))


# --------------------------------------------------------------- numerics
def _matmul_pair(xl, x, yl, y, outl):
    """Same math as einsum without the 52-label limit (batch/M/N/K grouping)."""
    xs, ys, os_ = set(xl), set(yl), set(outl)
    bl = [l for l in xl if l in ys and l in os_]
    kl = [l for l in xl if l in ys and l not in os_]
    ml = [l for l in xl if l not in ys and l in os_]
    nl = [l for l in yl if l not in xs and l in os_]
    # dangling (single-operand, summed) labels
    xd = [l for l in xl if l not in ys and l not in os_]
    yd = [l for l in yl if l not in xs and l not in os_]
    if xd:
        x = x.sum(axis=tuple(xl.index(l) for l in xd))
        xl = [l for l in xl if l not in xd]
    if yd:
        y = y.sum(axis=tuple(yl.index(l) for l in yd))
        yl = [l for l in yl if l not in yd]
    dim = {}
    for l, s in zip(xl, x.shape):
        dim[l] = s
    for l, s in zip(yl, y.shape):
        dim[l] = s
    pr = lambda ls: int(np.prod([dim[l] for l in ls], dtype=np.int64)) if ls else 1
    xa = np.transpose(x, [xl.index(l) for l in bl + ml + kl]).reshape(pr(bl), pr(ml), pr(kl))
    ya = np.transpose(y, [yl.index(l) for l in bl + kl + nl]).reshape(pr(bl), pr(kl), pr(nl))
    z = np.matmul(xa, ya).reshape([dim[l] for l in bl + ml + nl])
    cur = bl + ml + nl
    return np.transpose(z, [cur.index(l) for l in outl]) if cur != list(outl) else z


def pairwise_contract(xl, x, yl, y, keep):
    """The reference's ``pairwise_contract`` (dense.py:61-76) on labelled
    arrays; the restated matmul form only past its 52-label limit."""
    if len(set(xl) | set(yl)) <= len(_LETTERS):
        t = _rd.pairwise_contract(_rd.DenseTensor(xl, x), _rd.DenseTensor(yl, y), keep)
        return tuple(t.labels), t.array
    for i, lbl in enumerate(xl):
        if lbl in yl and x.shape[i] != y.shape[yl.index(lbl)]:
            raise ValueError(f"dim mismatch on shared index {lbl}")
    outl = [l for l in xl if l in keep]
    outl += [l for l in yl if l in keep and l not in xl]
    return tuple(outl), _matmul_pair(list(xl), x, list(yl), y, outl)


def fix_index(labels, arr, label, value):
    """The reference's ``fix_index`` (dense.py:161-170)."""
    t = _rd.fix_index(_rd.DenseTensor(labels, arr), label, value)
    return tuple(t.labels), t.array


def slice_digits(dims, s):
    digits = []
    for w in reversed(dims):
        digits.append(s % w)
        s //= w
    return tuple(reversed(digits))


def contract_one(tn, tree, sliced=(), assignment=None, strip_exponent=False,
                 terms=None, record=None):
    """Contract one slice.  Returns (root array in output order, exponent10,
    op_count, peak_elements)."""
    if any(nd.data is None for nd in tn.nodes):
        raise ValueError("contract needs dense data on every node")
    terms = vertex_terms(tn, tree) if terms is None else terms
    S = tuple(sliced)
    assignment = assignment or {}
    by_id = {nd.id: nd for nd in tn.nodes}
    n = len(tree.leaves)
    buf = [None] * (2 * n - 1 if n > 1 else 1)
    exp10 = 0.0
    for i, nid in enumerate(tree.leaves):
        nd = by_id[nid]
        labels, arr = tuple(nd.indices), nd.data
        for lbl in S:
            if lbl in labels:
                labels, arr = fix_index(labels, arr, lbl, assignment[lbl])
        buf[i] = (labels, arr)
    ops, peak = 0, 0
    Sset = set(S)
    for k, (a, b) in enumerate(tree.pairs):
        v = n + k
        keep = set(terms[v]) - Sset
        xl, x = buf[a]
        yl, y = buf[b]
        u = set(xl) | set(yl)
        mac = 1
        for lbl in u:
            mac *= tn.index_table[lbl]
        ops += mac
        outl, z = pairwise_contract(xl, x, yl, y, keep)
        if strip_exponent:
            m = float(np.max(np.abs(z))) if z.size else 0.0
            if m > 0.0 and np.isfinite(m):
                e = math.floor(math.log10(m))
                z = z / (10.0 ** e)
                exp10 += e
        if not np.all(np.isfinite(z)):
            raise FloatingPointError(f"non-finite intermediate at vertex {v}")
        peak = max(peak, z.size)
        buf[a] = buf[b] = None
        buf[v] = (outl, z)
        if record is not None:
            record[v] = (outl, z)
    rl, r = buf[tree.root]
    out = [l for l in tn.output]
    # single-leaf tree: sum labels not in the output (nested-sum definition)
    extra = [l for l in rl if l not in out]
    if extra:
        r = r.sum(axis=tuple(rl.index(l) for l in extra))
        rl = tuple(l for l in rl if l not in extra)
    r = _rd.DenseTensor(rl, r).transpose_to(out).array
    return np.asarray(r, dtype=np.complex128), exp10, ops, peak


class _Kahan:
    def __init__(self, shape):
        self.s = np.zeros(shape, dtype=np.complex128)
        self.c = np.zeros(shape, dtype=np.complex128)

    def add(self, x):
        y = x - self.c
        t = self.s + y
        self.c = (t - self.s) - y
        self.s = t


def contract_sliced(tn, tree, sliced=(), slice_ids=None, strip_exponent=False):
    """Sum of per-slice contractions.

    Returns (value-or-open-tensor, exponent10, op_count).  ``slice_ids``
    restricts the sum to a subset (prefix runs / per-slice parity).
    """
    S = tuple(sliced)
    for lbl in S:
        if lbl in tn.output:
            raise ValueError(f"output label {lbl} cannot be sliced")
    dims = [tn.index_table[l] for l in S]
    d = int(np.prod(dims, dtype=object)) if dims else 1
    ids = range(d) if slice_ids is None else slice_ids
    terms = vertex_terms(tn, tree)
    acc = None
    total_ops = 0
    exps = []
    parts = []
    for s in ids:
        assign = dict(zip(S, slice_digits(dims, int(s))))
        r, e, ops, _ = contract_one(tn, tree, S, assign, strip_exponent, terms)
        total_ops += ops
        if strip_exponent:
            parts.append((r, e))
        else:
            if acc is None:
                acc = _Kahan(r.shape)
            acc.add(r)
    if strip_exponent:
        emax = max(e for _, e in parts)
        acc = _Kahan(parts[0][0].shape)
        for r, e in parts:
            acc.add(r * 10.0 ** (e - emax))
        val = acc.s
        exp10 = emax + tn.norm_exponent
    else:
        val = acc.s
        exp10 = 0.0
        if tn.norm_exponent:
            exp10 = tn.norm_exponent
    if val.ndim == 0:
        val = complex(val)
    return val, exp10, total_ops


def contract(tn, tree, strip_exponent=False):
    """Unsliced contraction."""
    return contract_sliced(tn, tree, (), None, strip_exponent)


def brute_force(tn):
    """Direct nested summation via one einsum over the whole network
    (acceptance criterion 2) -- small networks only."""
    labels = list(tn.index_table)
    if len(labels) > 52:
        raise ValueError("brute force limited to 52 labels")
    sym = {l: _LETTERS[i] for i, l in enumerate(labels)}
    subs = ",".join("".join(sym[l] for l in nd.indices) for nd in tn.nodes)
    sub = subs + "->" + "".join(sym[l] for l in tn.output)
    return np.einsum(sub, *[nd.data for nd in tn.nodes], optimize="greedy")
