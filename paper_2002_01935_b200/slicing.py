"""Index slicing: ``SliceSet``, ``sliced_metrics``, ``greedy_slice`` and the
canonical slice-id enumeration.

The reference specifies but does not implement the slicer
(`/root/reference/SPEC.md:463-508`); this module follows that spec:

* ``SliceSet`` fields labels / d / Ws / Cs and its JSON
  form ``{"labels", "d", "Ws", "log10_Cs"}``.
* ``sliced_metrics(tree, tn, S) -> (W_s, C_s)``: Eqs. (3)/(6) with S deleted
  from every incidence set, C_s = d * per-slice cost.
  Output labels may not be sliced.
* ``greedy_slice``: add the single label that minimises the resulting C_s
  among labels of width-achieving vertices until W_s <= target; restarts
  with multiplicative +-noise on the score keep the cheapest feasible set
  (PAPER.md:684-687).

Slice enumeration (the reference leaves it undefined):
slice id s in [0, d) maps to the mixed-radix digits of s over the SliceSet
label order, LAST label fastest -- identical to ``itertools.product`` order
and ``numpy.unravel_index(s, dims)``.  Per-GPU ranges are contiguous.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .refpkg import annotate_incidence

__all__ = ["SliceSet", "sliced_metrics", "sliced_cost_terms", "greedy_slice",
           "slice_assignment", "slice_digits", "iter_slice_assignments"]


@dataclass(frozen=True)
class SliceSet:
    labels: tuple
    d: int
    Ws: float
    Cs: int = field(default=0)
    per_slice_cost: int = field(default=0)

    @property
    def log10_Cs(self):
        return math.log10(self.Cs) if self.Cs > 0 else float("-inf")

    def to_dict(self):
        return {"labels": list(self.labels), "d": int(self.d), "Ws": self.Ws,
                "log10_Cs": self.log10_Cs}

    @classmethod
    def from_labels(cls, tree, tn, labels):
        labels = tuple(labels)
        ws, cs, per, d = _sliced(tree, tn, labels)
        return cls(labels, d, ws, cs, per)

    @classmethod
    def from_dict(cls, obj, tree, tn):
        ss = cls.from_labels(tree, tn, obj["labels"])
        if "d" in obj and int(obj["d"]) != ss.d:
            raise ValueError(f"slice set d={obj['d']} does not match labels (d={ss.d})")
        return ss


def _mask_product(mask, dims, all_two):
    if all_two:
        return 1 << bin(mask).count("1")
    p, i = 1, 0
    while mask:
        if mask & 1:
            p *= dims[i]
        mask >>= 1
        i += 1
    return p


class _MaskView:
    """Bit-mask form of an annotated tree (label id i <-> bit i)."""

    def __init__(self, tree, tn):
        annotate_incidence(tree, tn)
        ann = tree._ann
        alg = ann.view
        self.alg = alg
        self.n = tree.n
        self.dims = alg.dims
        self.all_two = all(d == 2 for d in alg.dims)
        masks = []
        for t in ann.counts:
            m = 0
            for li in t:
                m |= 1 << li
            masks.append(m)
        self.vmask = masks
        self.umask = [masks[a] | masks[b] for a, b in tree.pairs]
        self.out_mask = 0
        for lbl in tn.output:
            self.out_mask |= 1 << alg.label_ids[lbl]

    def to_mask(self, labels):
        m = 0
        for lbl in labels:
            if lbl not in self.alg.label_ids:
                raise ValueError(f"unknown sliced label {lbl}")
            m |= 1 << self.alg.label_ids[lbl]
        return m


def _sliced(tree, tn, labels):
    mv = _MaskView(tree, tn)
    if len(set(labels)) != len(labels):
        raise ValueError("repeated label in slice set")
    smask = mv.to_mask(labels)
    if smask & mv.out_mask:
        bad = [lbl for lbl in labels if lbl in tn.output][0]
        raise ValueError(f"output label {bad} cannot be sliced")
    d = 1
    for lbl in labels:
        d *= tn.index_table[lbl]
    if tree.n == 1:
        out = 1
        for lbl in tn.output:
            out *= tn.index_table[lbl]
        return math.log2(out), 0, 0, d
    keep = ~smask
    per = sum(_mask_product(u & keep, mv.dims, mv.all_two) for u in mv.umask)
    n = mv.n
    peak = max(_mask_product(m & keep, mv.dims, mv.all_two) for m in mv.vmask[n:])
    return (math.log2(peak) if peak > 0 else 0.0), d * per, per, d


def sliced_metrics(tree, tn, s_sliced):
    """(W_s, C_s) of ``tree`` with labels ``s_sliced`` summed last
    (SPEC.md:474-482)."""
    ws, cs, _, _ = _sliced(tree, tn, tuple(s_sliced))
    return ws, cs


def sliced_cost_terms(tree, tn, s_sliced):
    """Per-internal-vertex MAC counts U_v for one slice (exact ints)."""
    mv = _MaskView(tree, tn)
    keep = ~mv.to_mask(s_sliced)
    return {mv.n + k: _mask_product(u & keep, mv.dims, mv.all_two)
            for k, u in enumerate(mv.umask)}


def greedy_slice(tree, tn, target_Ws, restarts=8, noise=0.05, seed=0):
    """Greedy slice-set search to reach ``W_s <= target_Ws``."""
    mv = _MaskView(tree, tn)
    alg = mv.alg
    leaf_log2 = 0.0
    for nd in tn.nodes:
        leaf_log2 = max(leaf_log2, sum(math.log2(tn.index_table[lbl]) for lbl in nd.indices))
    if target_Ws < leaf_log2 - 1e-12:
        raise ValueError(f"target W_s={target_Ws} is smaller than the largest leaf "
                         f"tensor (log2 size {leaf_log2})")
    if tree.n == 1:
        return SliceSet.from_labels(tree, tn, ())
    n = mv.n
    dims = mv.dims
    rng = np.random.default_rng(seed)
    best = None
    for rep in range(max(1, restarts)):
        amp = 0.0 if rep == 0 else noise
        chosen, smask = [], 0
        while True:
            keep = ~smask
            sizes = [_mask_product(m & keep, dims, mv.all_two) for m in mv.vmask[n:]]
            peak = max(sizes)
            if math.log2(peak) <= target_Ws + 1e-12:
                break
            pool = 0
            for v, sz in enumerate(sizes):
                if sz == peak:
                    pool |= mv.vmask[n + v]
            pool &= keep & ~mv.out_mask
            if not pool:
                raise ValueError("no sliceable label left in the width-achieving vertices")
            terms = [_mask_product(u & keep, dims, mv.all_two) for u in mv.umask]
            base = sum(terms)
            cands = []
            li = 0
            m = pool
            while m:
                if m & 1:
                    cands.append(li)
                m >>= 1
                li += 1
            scored = []
            for li in cands:
                bit = 1 << li
                hit = 0
                for u, t in zip(mv.umask, terms):
                    if u & bit:
                        hit += t
                w = dims[li]
                cs = w * base - (w - 1) * hit  # d-relative C_s after adding li
                score = float(cs)
                if amp > 0.0:
                    score *= 1.0 + amp * rng.uniform(-1.0, 1.0)
                scored.append((score, cs, li))
            scored.sort(key=lambda t: (t[0], t[2]))
            li = scored[0][2]
            chosen.append(alg.labels[li])
            smask |= 1 << li
        cand = SliceSet.from_labels(tree, tn, chosen)
        if best is None or cand.Cs < best.Cs:
            best = cand
    return best


# --------------------------------------------------------------- enumeration
def slice_digits(dims, s):
    """Mixed-radix digits of slice id ``s`` (last dim fastest)."""
    s = int(s)
    total = 1
    for w in dims:
        total *= int(w)
    if not 0 <= s < total:
        raise ValueError(f"slice id {s} out of range [0, {total})")
    digits = [0] * len(dims)
    for i in range(len(dims) - 1, -1, -1):
        w = int(dims[i])
        digits[i] = s % w
        s //= w
    return tuple(digits)


def slice_assignment(tn, slice_set, s):
    """Slice id -> {label: value}."""
    labels = slice_set.labels if hasattr(slice_set, "labels") else tuple(slice_set)
    dims = [tn.index_table[lbl] for lbl in labels]
    return dict(zip(labels, slice_digits(dims, s)))


def iter_slice_assignments(tn, slice_set, start=0, stop=None):
    labels = slice_set.labels if hasattr(slice_set, "labels") else tuple(slice_set)
    dims = [tn.index_table[lbl] for lbl in labels]
    d = 1
    for w in dims:
        d *= w
    stop = d if stop is None else min(stop, d)
    for s in range(start, stop):
        yield dict(zip(labels, slice_digits(dims, s)))


def auto_slice(tree, tn, device_bytes, ws_max=None, ws_min=None, fill=0.9, restarts=2, seed=0,
               precision="3xtf32"):
    """HBM-aware slicing: the largest target W_s whose
    compiled plan -- the library's own arena plan (intermediates, GEMM operand
    planes, split-K partials), persistent hoisted tensors and leaves -- fits in
    ``fill * device_bytes``.  Larger W_s means fewer, larger slices and a lower
    total cost C_s.  Returns (SliceSet, plan_bytes)."""
    from .executor import SlicedPlan
    from .refpkg import metrics
    m = metrics(tree, tn)
    hi = int(math.floor(m.width if ws_max is None else min(ws_max, m.width)))
    lo = int(ws_min) if ws_min is not None else 1
    for ws in range(hi, lo - 1, -1):
        try:
            ss = greedy_slice(tree, tn, ws, restarts=restarts, seed=seed) if ws < m.width else \
                SliceSet.from_labels(tree, tn, ())
        except ValueError:
            break
        plan = SlicedPlan(tn, tree, ss, precision=precision)
        try:
            st = plan.stats()
            need = st["work_arena_bytes"] + st["persistent_bytes"] + st["leaf_bytes"]
        finally:
            plan.close()
        if st["peak_elements"] < (1 << 40) and need <= fill * device_bytes:
            return ss, need
    raise ValueError("no slice width fits the device memory")
