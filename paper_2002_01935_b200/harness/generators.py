"""Seeded network builders for the five BASELINE.json configurations.

Benchmark HARNESS, not product: the reference specifies generators
(`/root/reference/SPEC.md:560-636`) but ships none, and tier scope keeps them
out of the product.  The executor only needs networks of the right shape:

* ``random_regular(n, k)``        -- configuration model with rejection of
  loops / multi-edges plus a connectivity retry.
* ``square_lattice(L)``           -- vertex-form OBC/PBC lattice.
* ``grid_circuit(rows, cols, depth)`` -- GRCS-style (1+d+1) circuit amplitude
  <x|U|0^N>: Hadamard layer, 8 cycling CZ patterns, random {T, sqrt X,
  sqrt Y} single-qubit gates, Hadamard layer; every CZ spatially decomposed
  (chi = 2, Eq. 16) and then rank-simplified (rank<=2
  tensors absorbed into a neighbour) so that the network is made of rank-3
  tensors (BASELINE.json configs[3]: 742 rank-3 tensors at 7x7, d=40).
* ``sycamore_circuit(m)``          -- 53-qubit Sycamore-like lattice, ABCDCDAB
  coupler cycling, synthetic fSim(theta, phi) gates left undecomposed (rank 4).
* ``random_hyper_network``         -- small random hypergraph networks with
  hyperedges, open outputs and dims 1..3 for property tests.

Scaled random data: entries ~ CN(0,1) * 2^(-rank/4) so that E|value|^2 = 1
for closed dim-2 networks (SURVEY.md §8(d) synthetic inputs).
"""

from __future__ import annotations

import math

import numpy as np

from ..refpkg import TensorNetwork, TensorNode

__all__ = ["random_regular_graph", "random_regular", "square_lattice",
           "grid_circuit", "sycamore_circuit", "random_hyper_network",
           "graph_network", "circuit_statevector_amplitude"]


def _cnormal(rng, shape):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)


def random_regular_graph(n, k, seed):
    if (n * k) % 2 or k >= n:
        raise ValueError(f"no simple {k}-regular graph on {n} vertices")
    rng = np.random.default_rng(seed)
    for _ in range(10000):
        stubs = np.repeat(np.arange(n), k)
        rng.shuffle(stubs)
        edges = set()
        ok = True
        for i in range(0, len(stubs), 2):
            a, b = int(stubs[i]), int(stubs[i + 1])
            if a == b:
                ok = False
                break
            e = (min(a, b), max(a, b))
            if e in edges:
                ok = False
                break
            edges.add(e)
        if not ok:
            continue
        adj = {v: [] for v in range(n)}
        for a, b in edges:
            adj[a].append(b)
            adj[b].append(a)
        seen, stack = {0}, [0]
        while stack:
            v = stack.pop()
            for w in adj[v]:
                if w not in seen:
                    seen.add(w)
                    stack.append(w)
        if len(seen) == n:
            return sorted(edges)
    raise RuntimeError("failed to sample a connected regular graph")


def graph_network(n, edges, dim=2, seed=0, scaled=True):
    """One tensor per vertex, one label per edge (vertex form)."""
    rng = np.random.default_rng(seed + 7919)
    inc = {v: [] for v in range(n)}
    table = {}
    for i, (a, b) in enumerate(edges):
        lbl = f"e{i}"
        table[lbl] = dim
        inc[a].append(lbl)
        inc[b].append(lbl)
    nodes = []
    for v in range(n):
        labels = inc[v]
        shape = tuple(dim for _ in labels)
        data = _cnormal(rng, shape)
        if scaled:
            data = data * dim ** (-len(labels) / 4.0)
        nodes.append(TensorNode(v, labels, data))
    return TensorNetwork(nodes, table, ())


def random_regular(n, k, dim=2, seed=0):
    return graph_network(n, random_regular_graph(n, k, seed), dim, seed)


def square_lattice(L, boundary="open", dim=2, seed=0):
    if L < 2:
        raise ValueError("L >= 2 required")
    edges = []
    idx = lambda r, c: r * L + c
    for r in range(L):
        for c in range(L):
            if c + 1 < L:
                edges.append((idx(r, c), idx(r, c + 1)))
            elif boundary == "periodic":
                edges.append((idx(r, c), idx(r, 0)))
            if r + 1 < L:
                edges.append((idx(r, c), idx(r + 1, c)))
            elif boundary == "periodic":
                edges.append((idx(r, c), idx(0, c)))
    return graph_network(L * L, edges, dim, seed)


# ------------------------------------------------------------------ circuits
_SQ = {
    "T": np.array([[1, 0], [0, np.exp(1j * np.pi / 4)]], dtype=np.complex128),
    "SX": 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]], dtype=np.complex128),
    "SY": 0.5 * np.array([[1 + 1j, -1 - 1j], [1 + 1j, 1 + 1j]], dtype=np.complex128),
    "SW": None,  # filled below: sqrt of (X+Y)/sqrt2
    "H": np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2.0),
}
_W = (np.array([[0, 1], [1, 0]]) + np.array([[0, -1j], [1j, 0]])) / math.sqrt(2.0)
_evals, _evecs = np.linalg.eigh(_W)
_SQ["SW"] = (_evecs @ np.diag(np.sqrt(_evals.astype(np.complex128))) @ _evecs.conj().T)


def _cz_halves():
    """CZ = sum_k A[o1,i1,k] B[o2,i2,k]  (chi = 2 spatial split, Eq. 16)."""
    A = np.zeros((2, 2, 2), dtype=np.complex128)
    B = np.zeros((2, 2, 2), dtype=np.complex128)
    for i in range(2):
        A[i, i, i] = 1.0
        B[i, i, 0] = 1.0
        B[i, i, 1] = (-1.0) ** i
    return A, B


def _fsim(theta, phi):
    c, s = math.cos(theta), math.sin(theta)
    U = np.zeros((4, 4), dtype=np.complex128)
    U[0, 0] = 1.0
    U[1, 1] = c
    U[1, 2] = -1j * s
    U[2, 1] = -1j * s
    U[2, 2] = c
    U[3, 3] = np.exp(-1j * phi)
    return U.reshape(2, 2, 2, 2)  # (o1, o2, i1, i2)


class _CircuitTN:
    """Wire-by-wire circuit network builder with rank simplification."""

    def __init__(self, nq):
        self.nq = nq
        self.tensors = []      # list of [labels(list), data]
        self.wire = []
        self.nlab = 0
        for q in range(nq):
            lbl = self._new()
            self.wire.append(lbl)
            self.tensors.append([[lbl], np.array([1.0, 0.0], dtype=np.complex128)])

    def _new(self):
        self.nlab += 1
        return f"x{self.nlab - 1}"

    def gate1(self, q, U):
        o = self._new()
        self.tensors.append([[o, self.wire[q]], U.copy()])
        self.wire[q] = o

    def cz(self, q1, q2):
        A, B = _cz_halves()
        o1, o2, k = self._new(), self._new(), self._new()
        self.tensors.append([[o1, self.wire[q1], k], A])
        self.tensors.append([[o2, self.wire[q2], k], B])
        self.wire[q1], self.wire[q2] = o1, o2

    def gate1_diag(self, q, U):
        """Diagonal single-qubit gate, diagonal-reduced: a
        rank-1 node on the wire label, which is not advanced (hyperedge)."""
        self.tensors.append([[self.wire[q]], np.diag(U).copy()])

    def cz_diag(self, q1, q2):
        """CZ diagonal-reduced: rank-2 node M[a, b] = (-1)^(a b) on the two
        wire labels, which continue as hyperedges."""
        M = np.array([[1.0, 1.0], [1.0, -1.0]], dtype=np.complex128)
        self.tensors.append([[self.wire[q1], self.wire[q2]], M])

    def gate2(self, q1, q2, U4):
        o1, o2 = self._new(), self._new()
        self.tensors.append([[o1, o2, self.wire[q1], self.wire[q2]], U4.copy()])
        self.wire[q1], self.wire[q2] = o1, o2

    def close(self, bitstring):
        for q in range(self.nq):
            v = np.zeros(2, dtype=np.complex128)
            v[int(bitstring[q])] = 1.0
            self.tensors.append([[self.wire[q]], v])

    def simplify(self, hyper=False):
        """Absorb every rank<=2 tensor into its highest-rank neighbour.  With
        hyperedges (diagonal-reduced circuits) only into a neighbour that
        already carries all its labels, so no rank grows (rank-simplification,
        PAPER.md §III.G)."""
        ts = [t for t in self.tensors]
        alive = list(range(len(ts)))
        holders = {}
        for i, (labels, _) in enumerate(ts):
            for lbl in labels:
                holders.setdefault(lbl, set()).add(i)
        changed = True
        while changed:
            changed = False
            for i in list(alive):
                if ts[i] is None or len(ts[i][0]) > 2:
                    continue
                labels = ts[i][0]
                nbrs = set()
                for lbl in labels:
                    nbrs |= holders[lbl]
                nbrs.discard(i)
                if hyper:
                    nbrs = {t for t in nbrs if set(labels) <= set(ts[t][0])}
                if not nbrs:
                    continue
                j = max(nbrs, key=lambda t: (len(ts[t][0]), -t))
                la, A = ts[i]
                lb, B = ts[j]
                shared = [l for l in la if l in lb]
                # a shared label carried by other tensors too (hyperedge) stays
                # as a batch label; only labels private to i and j are summed
                summed = [l for l in shared if holders[l] <= {i, j}]
                outl = [l for l in lb if l not in summed] + [l for l in la if l not in summed and l not in lb]
                sym = {}
                for l in la + lb:
                    sym.setdefault(l, chr(97 + len(sym)))
                sub = "{},{}->{}".format("".join(sym[l] for l in la), "".join(sym[l] for l in lb),
                                         "".join(sym[l] for l in outl))
                C = np.einsum(sub, A, B)
                for l in la:
                    holders[l].discard(i)
                for l in lb:
                    holders[l].discard(j)
                ts[j] = [outl, C]
                for l in outl:
                    holders[l].add(j)
                ts[i] = None
                alive.remove(i)
                changed = True
        self.tensors = [ts[i] for i in alive]

    def network(self):
        table, nodes = {}, []
        order = {}
        for labels, _ in self.tensors:
            for l in labels:
                order.setdefault(l, int(l[1:]))
        for l in sorted(order, key=order.get):
            table[l] = 2
        for nid, (labels, data) in enumerate(self.tensors):
            nodes.append(TensorNode(nid, labels, data))
        return TensorNetwork(nodes, table, ())


_PATTERNS = [("H", 0, 0), ("H", 1, 1), ("V", 0, 0), ("V", 1, 1),
             ("H", 1, 0), ("H", 0, 1), ("V", 1, 0), ("V", 0, 1)]


def _grid_layer(rows, cols, t):
    d, off, stag = _PATTERNS[t % 8]
    pairs = []
    if d == "H":
        for r in range(rows):
            if r % 2 != stag:
                continue
            for c in range(off, cols - 1, 2):
                pairs.append((r * cols + c, r * cols + c + 1))
    else:
        for c in range(cols):
            if c % 2 != stag:
                continue
            for r in range(off, rows - 1, 2):
                pairs.append((r * cols + c, (r + 1) * cols + c))
    return pairs


def _grid_ops(rows, cols, depth, seed):
    """Gate list of a GRCS-style (1+depth+1) circuit."""
    rng = np.random.default_rng(seed)
    nq = rows * cols
    ops = [("1", q, "H") for q in range(nq)]
    prev_cz = set()
    last = ["H"] * nq
    for t in range(depth):
        pairs = _grid_layer(rows, cols, t)
        busy = {q for p in pairs for q in p}
        for q in range(nq):
            if q in prev_cz and q not in busy:
                choices = [g for g in ("T", "SX", "SY") if g != last[q]]
                g = choices[int(rng.integers(len(choices)))]
                ops.append(("1", q, g))
                last[q] = g
        for a, b in pairs:
            ops.append(("cz", a, b))
        prev_cz = busy
    for q in range(nq):
        ops.append(("1", q, "H"))
    return nq, ops


def grid_circuit(rows, cols, depth, seed=0, bitstring=None, simplify=True, diag=False):
    """Amplitude network <x|U|0^N> of a GRCS-style rows x cols circuit.
    ``diag=True`` diagonal-reduces CZ and T gates (PAPER.md
    §III.G): their wires continue as hyperedges instead of being split, the
    hyperedge-heavy form the paper's JAX executor handled poorly."""
    nq, ops = _grid_ops(rows, cols, depth, seed)
    bitstring = "0" * nq if bitstring is None else bitstring
    if len(bitstring) != nq:
        raise ValueError("bitstring length mismatch")
    c = _CircuitTN(nq)
    for op in ops:
        if op[0] == "1":
            if diag and op[2] == "T":
                c.gate1_diag(op[1], _SQ[op[2]])
            else:
                c.gate1(op[1], _SQ[op[2]])
        elif diag:
            c.cz_diag(op[1], op[2])
        else:
            c.cz(op[1], op[2])
    c.close(bitstring)
    if simplify:
        c.simplify(hyper=diag)
    return c.network()


def circuit_statevector_amplitude(rows, cols, depth, seed=0, bitstring=None):
    """Dense statevector amplitude (small circuits only) -- test oracle for
    the generator itself."""
    nq, ops = _grid_ops(rows, cols, depth, seed)
    psi = np.zeros([2] * nq, dtype=np.complex128)
    psi[(0,) * nq] = 1.0
    cz = np.diag([1, 1, 1, -1]).astype(np.complex128).reshape(2, 2, 2, 2)
    for op in ops:
        if op[0] == "1":
            psi = np.moveaxis(np.tensordot(_SQ[op[2]], psi, axes=([1], [op[1]])), 0, op[1])
        else:
            a, b = op[1], op[2]
            psi = np.moveaxis(np.tensordot(cz, psi, axes=([2, 3], [a, b])), [0, 1], [a, b])
    bitstring = "0" * nq if bitstring is None else bitstring
    return psi[tuple(int(ch) for ch in bitstring)]


# Sycamore-53 qubit coordinates: 54 sites of a 9 x 12 checkerboard (a rotated
# 6 x 9 grid) minus one dead qubit.
def _sycamore_layout():
    qubits = [(r, c) for r in range(9) for c in range(12) if (r + c) % 2 == 0]
    assert len(qubits) == 54
    qubits.pop(3)  # dead qubit -> 53
    return qubits


def sycamore_circuit(m, seed=0, bitstring=None, simplify=True):
    """Sycamore-like 53-qubit amplitude, ABCDCDAB couplers, synthetic fSim
    gates kept rank-4 (no decomposition)."""
    rng = np.random.default_rng(seed)
    qs = _sycamore_layout()
    pos = {q: i for i, q in enumerate(qs)}
    nq = len(qs)
    # A/B: couplers along one lattice diagonal (even / odd rows), C/D: the
    # other diagonal -- each pattern is a matching; ABCDCDAB cycling
    groups = {"A": [], "B": [], "C": [], "D": []}
    for (r, c), i in pos.items():
        for dc, even, odd in ((1, "A", "B"), (-1, "C", "D")):
            nb = (r + 1, c + dc)
            if nb in pos:
                groups[even if r % 2 == 0 else odd].append((i, pos[nb]))
    order = "ABCDCDAB"
    circ = _CircuitTN(nq)
    last = [None] * nq
    for cyc in range(m):
        for q in range(nq):
            choices = [g for g in ("SX", "SY", "SW") if g != last[q]]
            g = choices[int(rng.integers(len(choices)))]
            circ.gate1(q, _SQ[g])
            last[q] = g
        for a, b in groups[order[cyc % 8]]:
            th = float(rng.uniform(0.3, 1.3))
            ph = float(rng.uniform(0.1, 0.7))
            circ.gate2(a, b, _fsim(th, ph))
    for q in range(nq):
        choices = [g for g in ("SX", "SY", "SW") if g != last[q]]
        circ.gate1(q, _SQ[choices[int(rng.integers(len(choices)))]])
    bitstring = "0" * nq if bitstring is None else bitstring
    circ.close(bitstring)
    if simplify:
        circ.simplify()
    return circ.network()


def random_hyper_network(n_nodes, n_labels, seed, max_rank=4, dims=(1, 2, 3),
                         p_output=0.3, p_hyper=0.3, with_data=True):
    """Small random hypergraph network: labels on 1..4 nodes, some outputs."""
    rng = np.random.default_rng(seed)
    table = {}
    holders = {v: [] for v in range(n_nodes)}
    labels = [f"l{i}" for i in range(n_labels)]
    for lbl in labels:
        table[lbl] = int(dims[int(rng.integers(len(dims)))])
        k = 2
        if rng.random() < p_hyper:
            k = int(rng.integers(1, 5))
        k = min(k, n_nodes)
        cand = [v for v in range(n_nodes) if len(holders[v]) < max_rank] or list(range(n_nodes))
        chosen = rng.choice(len(cand), size=min(k, len(cand)), replace=False)
        for c in chosen:
            holders[cand[int(c)]].append(lbl)
    for v in range(n_nodes):
        if not holders[v]:
            lbl = f"s{v}"
            table[lbl] = 2
            holders[v].append(lbl)
    used = [l for l in table if any(l in holders[v] for v in range(n_nodes))]
    table = {l: table[l] for l in used}
    output = [l for l in used if rng.random() < p_output][:4]
    rng.shuffle(output)
    nodes = []
    for v in range(n_nodes):
        labs = holders[v]
        shape = tuple(table[l] for l in labs)
        data = _cnormal(rng, shape) if with_data else None
        nodes.append(TensorNode(v, labs, data))
    return TensorNetwork(nodes, table, tuple(output))
