"""B200 executor: the drop-in for the reference's SPEC executor entry points.

* ``contract(tn, tree, options)`` -> (value-or-open-tensor, exponent10, op_count)
  (`/root/reference/SPEC.md:515-523`)
* ``contract_sliced(tn, tree, slice_set, options)`` -> same triple, summed over
  every slice assignment; ``slice_ids`` restricts the sum
  to a contiguous prefix/range (the paper's "first 100 slices" protocol,
  PAPER.md:758).
* ``amplitude(circuit_tn, bitstring, tree, ...)``: open
  output legs projected onto the bitstring (column projection) -- the same
  compiled plan is reused across bitstrings, only leaf data is re-bound.

Everything numeric runs in libtnx.so on the GPU (hand-written sm_100a CUDA);
this module only interns labels, owns the plan handle and converts results.
Errors mirror the reference: ``ValueError`` for tree/slice problems,
``DataError`` for network data problems, ``FloatingPointError`` for
non-finite results.
"""

from __future__ import annotations

import ctypes as C
import math
import threading

import numpy as np

from . import _native as nat
from .refpkg import DataError, TensorNetwork, TensorNode

__all__ = ["SlicedPlan", "contract", "contract_sliced", "amplitude", "AmplitudeEngine",
           "allreduce_plans", "PRECISIONS"]

PRECISIONS = {"fp32": nat.PREC_FP32, "3xtf32": nat.PREC_3XTF32, "tf32-bf16x": nat.PREC_TF32_BF16X}
DEFAULT_PRECISION = "3xtf32"


def _precision(p):
    import os
    return p if p is not None else os.environ.get("TNX_PRECISION", DEFAULT_PRECISION)


def _as_labels(slice_set):
    if slice_set is None:
        return ()
    if hasattr(slice_set, "labels"):
        return tuple(slice_set.labels)
    return tuple(slice_set)


def _i32(values):
    arr = (C.c_int32 * max(1, len(values)))(*values)
    return arr


class SlicedPlan:
    """A compiled (network, tree, slice set) on one CUDA device.

    Compilation (bookkeeping, kernel selection, HBM arena plan) happens in
    libtnx at construction; ``bind`` uploads leaf data, precomputes the
    slice-invariant subtrees and captures the per-slice CUDA graph; ``run``
    contracts a slice range into the device accumulator.
    """

    def __init__(self, tn, tree, slice_set=(), device=0, precision=None, graph=True,
                 hoist=True, gemm_min_macs=0.0, tiled_pack=True, direct_planes=True,
                 strip_exponent=False):
        lib = nat.load()
        self.tn = tn
        self.tree = tree
        self.device = int(device)
        self.sliced = _as_labels(slice_set)
        if sorted(tree.leaves) != sorted(tn.node_ids):
            raise ValueError("tree leaves do not match network node ids")
        labels = list(tn.index_table)
        self.labels = labels
        lid = {l: i for i, l in enumerate(labels)}
        self.label_ids = lid
        for lbl in self.sliced:
            if lbl not in lid:
                raise ValueError(f"unknown sliced label {lbl}")
        ranks, leaf_labels = [], []
        for nid in tree.leaves:
            nd = tn.node(nid)
            for lbl in nd.indices:
                if lbl not in lid:
                    raise DataError(f"unknown index {lbl}@node{nd.id}")
            ranks.append(len(nd.indices))
            leaf_labels.extend(lid[l] for l in nd.indices)
        pairs = [c for p in tree.pairs for c in p]
        for lbl in tn.output:
            if lbl not in lid:
                raise DataError(f"unknown output index {lbl}")
        self._keep = dict(
            dims=(C.c_int64 * max(1, len(labels)))(*[tn.index_table[l] for l in labels]),
            ranks=_i32(ranks), leaf_labels=_i32(leaf_labels), pairs=_i32(pairs),
            out=_i32([lid[l] for l in tn.output]), sl=_i32([lid[l] for l in self.sliced]))
        k = self._keep
        precision = _precision(precision)
        flags = ((0 if graph else nat.FLAG_NO_GRAPH) | (0 if hoist else nat.FLAG_NO_HOIST)
                 | (0 if tiled_pack else nat.FLAG_NO_TILED_PACK)
                 | (0 if direct_planes else nat.FLAG_NO_DIRECT)
                 | (nat.FLAG_STRIP_EXPONENT if strip_exponent else 0))
        self.strip_exponent = bool(strip_exponent)
        if precision not in PRECISIONS:
            raise ValueError(f"unknown precision {precision!r}; choose from {sorted(PRECISIONS)}")
        self.precision = precision
        desc = nat.PlanDesc(len(labels), k["dims"], tree.n, k["ranks"], k["leaf_labels"], k["pairs"],
                            len(tn.output), k["out"], len(self.sliced), k["sl"],
                            PRECISIONS[precision], self.device, flags, 0, float(gemm_min_macs))
        handle = C.c_void_p()
        nat.check(lib.tnx_plan_create(C.byref(desc), C.byref(handle)))
        self._h = handle
        self._lib = lib
        self._bound = False
        st = nat.Stats()
        nat.check(lib.tnx_stats_get(self._h, C.byref(st)))
        self._stats = st
        self.out_shape = tuple(tn.index_table[l] for l in tn.output)

    # ------------------------------------------------------------ properties
    @property
    def d(self):
        return self._stats.d_lo | (self._stats.d_hi << 64)

    @property
    def ops_per_slice(self):
        """Exact per-slice MAC count sum_v U_v (C_s / d)."""
        return self._stats.op_count_lo | (self._stats.op_count_hi << 64)

    @property
    def flops_per_slice(self):
        return 8 * self.ops_per_slice

    @property
    def width(self):
        return self._stats.width

    def stats(self):
        st = nat.Stats()
        nat.check(self._lib.tnx_stats_get(self._h, C.byref(st)))
        self._stats = st
        s = st
        return {"op_count_per_slice": self.ops_per_slice, "d": self.d, "W_s": s.width,
                "peak_elements": s.peak_elements, "work_arena_bytes": s.work_arena_bytes,
                "persistent_bytes": s.persistent_bytes, "leaf_bytes": s.leaf_bytes,
                "num_vertices": s.num_vertices, "num_hoisted": s.num_hoisted,
                "num_gemm": s.num_gemm, "num_simt": s.num_simt,
                "launches_per_slice": s.launches_per_slice, "out_elements": s.out_elements}

    def vertex_info(self):
        out = []
        vi = nat.VertexInfo()
        for i in range(self._stats.num_vertices):
            nat.check(self._lib.tnx_vertex_info_get(self._h, i, C.byref(vi)))
            out.append({"ssa": vi.ssa, "kind": nat.KIND_NAMES[vi.kind], "hoisted": bool(vi.hoisted),
                        "rank": vi.rank, "m": vi.m, "n": vi.n, "k": vi.k, "batch": vi.batch,
                        "macs": vi.macs_lo | (vi.macs_hi << 64)})
        return out

    # ------------------------------------------------------------ execution
    def bind(self, tn=None, stream=None, leaf_arrays=None):
        """Upload leaf data (host complex128 from ``tn`` nodes, or a list of
        contiguous complex64/complex128 host arrays / CUDA torch tensors in
        SSA leaf order).  Every array must hold exactly the leaf's
        prod(dims) elements; a wrong size or dtype raises ``DataError``.
        CUDA tensors are read on torch's current stream of the plan's device
        unless ``stream`` is given."""
        tn = self.tn if tn is None else tn
        if leaf_arrays is None:
            arrs = []
            for nid in self.tree.leaves:
                nd = tn.node(nid)
                if nd.data is None:
                    raise ValueError(f"contract needs dense data on every node (node {nid})")
                arrs.append(np.ascontiguousarray(nd.data, dtype=np.complex128))
            leaf_arrays = arrs
        if len(leaf_arrays) != self.tree.n:
            raise DataError(f"{len(leaf_arrays)} leaf arrays for {self.tree.n} leaves")
        loc, dtype, ptrs, hold = self._leaf_pointers(leaf_arrays)
        if loc == nat.LOC_DEVICE and stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device)
        self._hold = hold
        nat.check(self._lib.tnx_bind_leaves(self._h, ptrs, dtype, loc, self._stream(stream)))
        self._bound = True
        return self

    def _leaf_sizes(self):
        sizes = getattr(self, "_sizes", None)
        if sizes is None:
            sizes = []
            for nid in self.tree.leaves:
                p = 1
                for lbl in self.tn.node(nid).indices:
                    p *= self.tn.index_table[lbl]
                sizes.append(p)
            self._sizes = sizes
        return sizes

    def _leaf_pointers(self, arrays):
        ptrs = (C.c_void_p * max(1, len(arrays)))()
        sizes = self._leaf_sizes()
        first = arrays[0]
        if hasattr(first, "is_cuda") and first.is_cuda:
            import torch
            dt = first.dtype
            if dt not in (torch.complex64, torch.complex128):
                raise DataError(f"leaf tensors must be complex64 or complex128, got {dt}")
            hold = []
            for i, a in enumerate(arrays):
                if not getattr(a, "is_cuda", False) or a.dtype != dt:
                    raise DataError(f"leaf {i}: all leaf tensors must be CUDA tensors of dtype {dt}")
                if a.device.index != self.device:
                    raise DataError(f"leaf {i} lives on cuda:{a.device.index}, plan on cuda:{self.device}")
                if a.numel() != sizes[i]:
                    raise DataError(f"leaf {i}: {a.numel()} elements, its labels need {sizes[i]}")
                c = a.contiguous()       # kept alive in `hold` until the next bind
                hold.append(c)
                ptrs[i] = c.data_ptr()
            dtype = nat.DTYPE_C64 if dt == torch.complex64 else nat.DTYPE_C128
            return nat.LOC_DEVICE, dtype, ptrs, hold
        # re-binding the same (contiguous, right-dtype) host arrays -- new values in
        # the same buffers, e.g. one bind per bitstring or per step -- reuses the
        # marshalled pointer table; the library still copies the data every bind
        cache = getattr(self, "_ptr_cache", None)
        if (cache is not None and len(cache[0]) == len(arrays)
                and all(a is b for a, b in zip(arrays, cache[0]))):
            return nat.LOC_HOST, cache[1], cache[2], cache[3]
        conv = []
        first = np.asarray(first)
        if not np.issubdtype(first.dtype, np.number):
            raise DataError(f"leaf arrays must be numeric, got {first.dtype}")
        dtype = nat.DTYPE_C64 if first.dtype == np.complex64 else nat.DTYPE_C128
        want = np.complex64 if dtype == nat.DTYPE_C64 else np.complex128
        reusable = True
        for i, a in enumerate(arrays):
            c = np.ascontiguousarray(a, dtype=want)
            if c.size != sizes[i]:
                raise DataError(f"leaf {i}: {c.size} elements, its labels need {sizes[i]}")
            reusable = reusable and c is a
            conv.append(c)
            ptrs[i] = c.__array_interface__["data"][0]
        self._ptr_cache = (list(arrays), dtype, ptrs, conv) if reusable else None
        return nat.LOC_HOST, dtype, ptrs, conv

    @staticmethod
    def _stream(stream):
        if stream is None:
            return None
        if isinstance(stream, int):
            return C.c_void_p(stream)
        return C.c_void_p(stream.cuda_stream)

    def run(self, s_begin=0, s_end=None, stream=None):
        if not self._bound:
            raise ValueError("bind() leaf data before run()")
        s_end = self.d if s_end is None else s_end
        nat.check(self._lib.tnx_run_slices(self._h, int(s_begin), int(s_end), self._stream(stream)))
        return self

    def run_ids(self, ids, stream=None):
        """Contract the slices in ``ids`` (an iterable of ids in [0, d), any
        order) into the accumulator in one library call (tnx_run_slice_ids)."""
        if not self._bound:
            raise ValueError("bind() leaf data before run_ids()")
        arr = (C.c_uint64 * max(1, len(ids)))(*[int(s) for s in ids])
        nat.check(self._lib.tnx_run_slice_ids(self._h, arr, len(ids), self._stream(stream)))
        return self

    def reset(self, stream=None):
        nat.check(self._lib.tnx_reset_accumulator(self._h, self._stream(stream)))

    def result(self, stream=None):
        n = int(self._stats.out_elements)
        buf = np.zeros(2 * max(n, 1), dtype=np.float64)
        nat.check(self._lib.tnx_partial_result(self._h, buf.ctypes.data_as(C.POINTER(C.c_double)), n,
                                               self._stream(stream)))
        val = (buf[0::2] + 1j * buf[1::2])[:n].reshape(self.out_shape)
        return val

    def result_async(self, out, stream=None):
        """Enqueue the accumulator's copy into ``out`` (a caller-owned buffer of
        2 * out_elements float64 -- pinned host memory, e.g. a pinned torch
        tensor -- given as an object with ``data_ptr()``, a numpy array or an
        address) and return at once; ``out`` holds the complex128 values once
        the stream is synchronised."""
        n = int(self._stats.out_elements)
        if hasattr(out, "data_ptr"):
            if out.numel() < 2 * max(n, 1):
                raise ValueError("result_async buffer too small")
            ptr = out.data_ptr()
        elif hasattr(out, "ctypes"):
            if out.size < 2 * max(n, 1):
                raise ValueError("result_async buffer too small")
            ptr = out.ctypes.data
        else:
            ptr = int(out)
        nat.check(self._lib.tnx_partial_result_async(self._h, C.c_void_p(ptr), n, self._stream(stream)))

    def profile_slice(self, s=0, with_bytes=False):
        """Per-launch CUDA-event timings of one (non-accumulated) slice:
        list of (kind, ssa vertex, ms[, algorithmic bytes])."""
        n = self.stats()["launches_per_slice"] + 8
        ty = (C.c_int32 * n)()
        vx = (C.c_int32 * n)()
        ms = (C.c_float * n)()
        by = (C.c_double * n)()
        cnt = C.c_int32()
        nat.check(self._lib.tnx_profile_slice(self._h, int(s), ty, vx, ms, by, n, C.byref(cnt)))
        names = {0: "gather", 1: "simt", 2: "pack", 3: "gemm", 4: "accum"}
        if with_bytes:
            return [(names[ty[i]], vx[i], float(ms[i]), float(by[i])) for i in range(cnt.value)]
        return [(names[ty[i]], vx[i], float(ms[i])) for i in range(cnt.value)]

    def result_exp(self, stream=None):
        """strip_exponent plans: (mantissas, base-2 exponents) per element."""
        n = int(self._stats.out_elements)
        buf = np.zeros(2 * max(n, 1), dtype=np.float64)
        ex = np.zeros(max(n, 1), dtype=np.int64)
        nat.check(self._lib.tnx_partial_result_exp(self._h, buf.ctypes.data_as(C.POINTER(C.c_double)),
                                                   ex.ctypes.data_as(C.POINTER(C.c_int64)), n,
                                                   self._stream(stream)))
        m = (buf[0::2] + 1j * buf[1::2])[:n].reshape(self.out_shape)
        return m, ex[:n].reshape(self.out_shape)

    def synchronize(self):
        nat.check(self._lib.tnx_synchronize(self._h))

    def debug_vertex(self, s, v):
        """Intermediate tensor of SSA vertex v for slice s: (labels, array)."""
        info = [x for x in self.vertex_info() if x["ssa"] == v]
        if not info:
            raise ValueError("vertex must be internal")
        rank = info[0]["rank"]
        # size from layout: query with a probe buffer
        lay = (C.c_int32 * max(1, rank))()
        rk = C.c_int32()
        size = self._vertex_size(v)
        buf = np.zeros(2 * size, dtype=np.float32)
        nat.check(self._lib.tnx_debug_vertex(self._h, int(s), int(v),
                                             buf.ctypes.data_as(C.POINTER(C.c_float)), size, lay,
                                             C.byref(rk)))
        labels = tuple(self.labels[lay[i]] for i in range(rk.value))
        shape = tuple(self.tn.index_table[l] for l in labels)
        return labels, (buf[0::2] + 1j * buf[1::2]).astype(np.complex64).reshape(shape)

    def _vertex_size(self, v):
        from .refpkg import ordered_labels
        size = 1
        S = set(self.sliced)
        for lbl in ordered_labels(self.tree, self.tn, v):
            if lbl not in S:
                size *= self.tn.index_table[lbl]
        return size

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.tnx_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def _combine_exp(parts, tn):
    """Sum of mantissa * 2^e parts -> (value, exponent10) without overflow."""
    logs = []
    for m, e in parts:
        m = np.asarray(m)
        with np.errstate(divide="ignore"):
            lm = np.where(m != 0, np.log10(np.abs(m)) + e * math.log10(2.0), -np.inf)
        logs.append(lm)
    top = max(float(np.max(lm)) if np.size(lm) else -np.inf for lm in logs)
    e10 = 0 if not np.isfinite(top) else math.floor(top)
    total = 0
    for m, e in parts:
        total = total + np.asarray(m) * np.power(10.0, np.asarray(e) * math.log10(2.0) - e10)
    arr = np.asarray(total)
    if not np.all(np.isfinite(arr)):
        raise FloatingPointError("non-finite contraction value")
    exp10 = e10 + tn.norm_exponent
    return (complex(arr) if arr.ndim == 0 else arr), exp10


def _finish(val, tn, strip_exponent):
    arr = np.asarray(val)
    if not np.all(np.isfinite(arr)):
        raise FloatingPointError("non-finite contraction value")
    exp10 = tn.norm_exponent
    if strip_exponent:
        m = float(np.max(np.abs(arr))) if arr.size else 0.0
        if m > 0.0:
            e = math.floor(math.log10(m))
            arr = arr / 10.0 ** e
            exp10 += e
    if arr.ndim == 0:
        return complex(arr), exp10
    return arr, exp10


def _slice_runs(d, slice_ids):
    """Slice ids to run, as contiguous [a, b) runs in the given order.

    ``None`` = every slice; a ``range`` with step 1 = one run; any other
    iterable is a list of slice ids (the oracle's meaning, duplicates summed
    twice), grouped into maximal consecutive runs."""
    if slice_ids is None:
        return [(0, d)]
    if isinstance(slice_ids, range):
        if slice_ids.step != 1:
            raise ValueError("a slice_ids range must have step 1 (pass a list for other id sets)")
        if not 0 <= slice_ids.start <= slice_ids.stop <= d:
            raise ValueError(f"slice range [{slice_ids.start}, {slice_ids.stop}) out of [0, {d})")
        return [(slice_ids.start, slice_ids.stop)] if slice_ids.stop > slice_ids.start else []
    runs = []
    for s in slice_ids:
        s = int(s)
        if not 0 <= s < d:
            raise ValueError(f"slice id {s} out of [0, {d})")
        if runs and runs[-1][1] == s:
            runs[-1][1] = s + 1
        else:
            runs.append([s, s + 1])
    return [(a, b) for a, b in runs]


def _split_runs(runs, G):
    """Split runs into G consecutive shares of (nearly) equal slice counts."""
    total = sum(b - a for a, b in runs)
    cuts = [total * g // G for g in range(G + 1)]
    shares = [[] for _ in range(G)]
    pos = 0
    for a, b in runs:
        for g in range(G):
            lo, hi = max(a, a + cuts[g] - pos), min(b, a + cuts[g + 1] - pos)
            if hi > lo:
                shares[g].append((lo, hi))
        pos += b - a
    return shares


def allreduce_plans(plans, streams=None):
    """Sum the accumulators of bound plans (one process, any devices) on the
    device through ``tnx_allreduce``; afterwards every plan holds the total."""
    plans = list(plans)
    if not plans:
        raise ValueError("no plans")
    lib = plans[0]._lib
    hs = (C.c_void_p * len(plans))(*[p._h.value if isinstance(p._h, C.c_void_p) else p._h for p in plans])
    sts = None
    if streams is not None:
        sts = (C.c_void_p * len(plans))(*[SlicedPlan._stream(s).value if s is not None else None
                                          for s in streams])
    nat.check(lib.tnx_allreduce(hs, len(plans), sts))


def contract_sliced(tn, tree, slice_set=(), options=None, *, slice_ids=None, devices=(0,),
                    precision=None, graph=True, hoist=True):
    """Sum over slice assignments of the per-slice contraction.

    Returns (value-or-open-tensor, exponent10, op_count) with op_count the
    exact MAC count executed (C_s for the full range).  ``slice_ids``
    restricts the sum: a step-1 ``range`` or a list of slice ids (see
    ``_slice_runs``).  ``devices`` splits the ids into contiguous per-device
    shares (one host thread per device) and sums the complex128 partials.
    """
    options = dict(options or {})
    strip = bool(options.get("strip_exponent", False))
    devices = list(devices)
    plans = [SlicedPlan(tn, tree, slice_set, device=d, precision=precision, graph=graph, hoist=hoist,
                        strip_exponent=strip)
             for d in devices]
    try:
        runs = _slice_runs(plans[0].d, slice_ids)
        G = len(plans)
        shares = _split_runs(runs, G)
        errs = [None] * G

        def work(g):
            try:
                p = plans[g]
                p.bind()
                for a, b in shares[g]:
                    p.run(a, b)
            except BaseException as exc:  # noqa: BLE001
                errs[g] = exc

        if G == 1:
            work(0)
        else:
            th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        for e in errs:
            if e is not None:
                raise e
        if G > 1:
            allreduce_plans(plans)
        ops = plans[0].ops_per_slice * sum(b - a for a, b in runs)
        if strip:
            val, exp10 = _combine_exp([plans[0].result_exp()], tn)
            return val, exp10, ops
        val, exp10 = _finish(plans[0].result(), tn, strip)
        return val, exp10, ops
    finally:
        for p in plans:
            p.close()


def contract(tn, tree, options=None, **kw):
    """Unsliced contraction."""
    return contract_sliced(tn, tree, (), options, **kw)


_OPEN = ("x", "X", "*")


def _project(tn, bitstring):
    """Fix the open legs (tn.output order) to the bitstring (column projection,
    SPEC.md:533-537).  Positions marked 'x' / '*' stay open: they become the
    projected network's output legs, in qubit order, so the contraction yields
    the 2^N_f amplitudes of the open qubits at once (PAPER.md N_f open qubits)."""
    if len(bitstring) != len(tn.output):
        raise ValueError(f"bitstring length {len(bitstring)} != {len(tn.output)} open legs")
    fix, keep = {}, []
    for lbl, b in zip(tn.output, bitstring):
        if b in _OPEN:
            keep.append(lbl)
            continue
        if not str(b).isdigit():
            raise ValueError(f"bitstring character {b!r} is neither a digit nor an open marker")
        fix[lbl] = int(b)
    nodes = []
    for nd in tn.nodes:
        data, labels = nd.data, list(nd.indices)
        if data is None:
            raise ValueError("amplitude needs dense data")
        for lbl in list(labels):
            if lbl in fix:
                ax = labels.index(lbl)
                if not 0 <= fix[lbl] < data.shape[ax]:
                    raise ValueError(f"bit {fix[lbl]} out of range for leg {lbl}")
                data = np.take(data, fix[lbl], axis=ax)
                labels.pop(ax)
        nodes.append(TensorNode(nd.id, labels, data))
    table = {l: d for l, d in tn.index_table.items() if l not in fix}
    return TensorNetwork(nodes, table, tuple(keep), tn.norm_exponent)


def _open_pattern(bitstring):
    return tuple(i for i, b in enumerate(bitstring) if b in _OPEN)


def _default_tree(tn, trials=4, seed=0):
    """Tree for ``amplitude`` when the caller gives none: the reference's own
    Boltzmann-greedy driver (``greedy_sample``, drivers/greedy.py:144-158),
    best of ``trials`` (alpha, tau) shots by (cost, width) -- path finding stays
    the reference's (north_star)."""
    from .refpkg import greedy_sample, metrics
    rng = np.random.default_rng(seed)
    best, best_key = None, None
    for t in range(max(1, trials)):
        alpha, tau = (1.0, 0.0) if t == 0 else (float(rng.uniform(0.0, 2.0)), float(rng.choice([0.0, 0.05])))
        tree = greedy_sample(tn, alpha, tau, seed + t)
        m = metrics(tree, tn)
        key = (m.cost, m.width)
        if best is None or key < best_key:
            best, best_key = tree, key
    return best


def _device_free_bytes(device):
    import torch
    free, _total = torch.cuda.mem_get_info(device)
    return free


class AmplitudeEngine:
    """One compiled plan reused across bitstrings (only leaf data changes,
    PAPER.md:530).  ``open_qubits`` (positions, or a pattern
    string with 'x' marks) selects legs left open: every call must then mark
    exactly those positions and returns the (2,)*N_f amplitude tensor.

    ``tree=None`` takes the reference's ``greedy_sample`` tree of the
    projected network; ``slice_set=None`` slices it to the largest W_s whose
    plan fits the device (``auto_slice``)."""

    def __init__(self, circuit_tn, tree=None, slice_set=(), device=0, precision=None, open_qubits=()):
        self.tn = circuit_tn
        if isinstance(open_qubits, str):
            open_qubits = _open_pattern(open_qubits)
        self.open = tuple(sorted(int(i) for i in open_qubits))
        n = len(circuit_tn.output)
        if any(not 0 <= i < n for i in self.open):
            raise ValueError(f"open qubit positions {self.open} out of range for {n} legs")
        base = "".join("x" if i in self.open else "0" for i in range(n))
        ptn = _project(circuit_tn, base)
        self.tree = _default_tree(ptn) if tree is None else tree
        if slice_set is None:
            from .slicing import auto_slice
            slice_set, _ = auto_slice(self.tree, ptn, _device_free_bytes(device), precision=_precision(precision))
        self.slice_set = slice_set
        self.plan = SlicedPlan(ptn, self.tree, slice_set, device=device, precision=precision)

    def __call__(self, bitstring):
        """c_x (or the open-qubit tensor), including the network's
        ``10**norm_exponent`` factor (network.py:55-58)."""
        if _open_pattern(bitstring) != self.open:
            raise ValueError(f"open positions of {bitstring!r} differ from the engine's {self.open}")
        ptn = _project(self.tn, bitstring)
        self.plan.bind(ptn)
        self.plan.run()
        val, exp10 = _finish(self.plan.result(), ptn, False)
        if exp10:
            val = val * 10.0 ** exp10
            if not np.all(np.isfinite(np.asarray(val))):
                raise FloatingPointError("amplitude overflows complex128 after applying norm_exponent")
        return val

    def close(self):
        self.plan.close()


def amplitude(circuit_tn, bitstring, tree=None, slice_set=None, **kw):
    """c_x = <x| U |0> of a circuit network whose open legs are the qubits
    (``amplitude(circuit_tn, bitstring) -> complex``).  The tree
    defaults to the reference's ``greedy_sample`` on the projected network and
    the slicing to the largest W_s that fits the device; 'x' / '*' in the
    bitstring leave that qubit open and return the amplitude tensor over the
    open qubits."""
    if len(bitstring) != len(circuit_tn.output):
        raise ValueError(f"bitstring length {len(bitstring)} != {len(circuit_tn.output)} open legs")
    eng = AmplitudeEngine(circuit_tn, tree, slice_set, open_qubits=_open_pattern(bitstring), **kw)
    try:
        return eng(bitstring)
    finally:
        eng.close()
