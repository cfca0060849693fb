"""Minimal tree sources for the harness (tests / bench on the GPU box).

Path finding is OUT OF SCOPE for this executor (north_star: "the Python
path-finding and hyper-optimization layer stays as the reference has it").
The benchmark trees for the large configurations are produced by the
reference's own drivers in the build container and committed as SSA path
files (``benchdata/``); this module only provides a small size-greedy
(alpha = 1, tau = 0 in the notation of drivers/greedy.py:1-11) and a
best-of-N randomised variant so tests can build trees for arbitrary random
networks where ``/root/reference`` does not exist.
"""

from __future__ import annotations

import heapq
import math

import numpy as np

from ..refpkg import ContractionTree, HyperView

__all__ = ["greedy_tree", "best_greedy_tree", "linear_tree"]


def _log2size(alg, term):
    return sum(math.log2(alg.dims[li]) for li in term)


def greedy_tree(tn, seed=0, temperature=0.0, alpha=1.0):
    """Agglomerative greedy: merge the adjacent pair with the smallest
    2^out - alpha (2^a + 2^b); optional Gumbel noise of scale ``temperature``
    on the log-score for randomised restarts."""
    alg = HyperView.from_network(tn)
    n = len(alg.terms)
    if n == 1:
        return ContractionTree(tn.node_ids, [])
    rng = np.random.default_rng(seed)
    terms = {i: alg.terms[i] for i in range(n)}
    lab2 = {}
    for i, t in terms.items():
        for li in t:
            lab2.setdefault(li, set()).add(i)
    nxt = n
    pairs = []
    heap = []

    def score(a, b):
        out = alg.merge_counts(terms[a], terms[b])
        s = 2.0 ** min(1000, _log2size(alg, out)) - alpha * (
            2.0 ** min(1000, _log2size(alg, terms[a])) + 2.0 ** min(1000, _log2size(alg, terms[b])))
        if temperature > 0:
            s = s - temperature * abs(s + 1.0) * float(rng.gumbel())
        return s

    def push_neighbors(f):
        seen = set()
        for li in terms[f]:
            for g in lab2.get(li, ()):
                if g != f and g not in seen:
                    seen.add(g)
                    a, b = (f, g) if f < g else (g, f)
                    heapq.heappush(heap, (score(a, b), a, b))

    for f in list(terms):
        push_neighbors(f)
    while len(terms) > 1:
        pick = None
        while heap:
            s, a, b = heapq.heappop(heap)
            if a in terms and b in terms:
                pick = (a, b)
                break
        if pick is None:  # disconnected: smallest two
            ks = sorted(terms, key=lambda f: (_log2size(alg, terms[f]), f))
            pick = (min(ks[0], ks[1]), max(ks[0], ks[1]))
        a, b = pick
        merged = alg.merge_counts(terms[a], terms[b])
        for f in (a, b):
            for li in terms[f]:
                lab2[li].discard(f)
            del terms[f]
        terms[nxt] = merged
        for li in merged:
            lab2.setdefault(li, set()).add(nxt)
        pairs.append((a, b))
        push_neighbors(nxt)
        nxt += 1
    return ContractionTree(tn.node_ids, pairs)


def best_greedy_tree(tn, trials=8, seed=0, target="cost"):
    from ..refpkg import metrics
    best, best_key = None, None
    for t in range(trials):
        tree = greedy_tree(tn, seed=seed + t, temperature=0.0 if t == 0 else 0.3)
        m = metrics(tree, tn)
        key = (m.cost, m.width) if target == "cost" else (m.width, m.cost)
        if best is None or key < best_key:
            best, best_key = tree, key
    return best


def linear_tree(tn):
    """Left-deep tree in node order (edge cases / tests)."""
    n = tn.num_nodes
    pairs = []
    cur = 0
    for i in range(1, n):
        pairs.append((cur, i))
        cur = n + i - 1
    return ContractionTree(tn.node_ids, pairs)
