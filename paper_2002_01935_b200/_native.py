"""ctypes binding of libtnx.so (C ABI declared in include/tnx.h).

The product path fails loudly when the library is missing: there is no CPU
fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtnx.so")

TNX_OK, TNX_ERR_INVALID, TNX_ERR_DATA, TNX_ERR_CUDA, TNX_ERR_OOM, TNX_ERR_NUMERIC, TNX_ERR_STATE = range(7)
PREC_FP32, PREC_3XTF32, PREC_TF32_BF16X = 0, 1, 2
DTYPE_C128, DTYPE_C64 = 0, 1
LOC_HOST, LOC_DEVICE = 0, 1
FLAG_NO_GRAPH, FLAG_NO_HOIST, FLAG_NO_TILED_PACK, FLAG_NO_DIRECT, FLAG_STRIP_EXPONENT = 1, 2, 4, 8, 16

KIND_NAMES = {0: "simt_thread", 1: "simt_warp", 2: "simt_split", 3: "gemm_tc", 4: "dot"}


class PlanDesc(C.Structure):
    _fields_ = [
        ("num_labels", C.c_int32), ("label_dims", C.POINTER(C.c_int64)),
        ("num_leaves", C.c_int32), ("leaf_ranks", C.POINTER(C.c_int32)),
        ("leaf_labels", C.POINTER(C.c_int32)), ("pairs", C.POINTER(C.c_int32)),
        ("num_output", C.c_int32), ("output_labels", C.POINTER(C.c_int32)),
        ("num_sliced", C.c_int32), ("sliced_labels", C.POINTER(C.c_int32)),
        ("precision", C.c_int32), ("device", C.c_int32), ("flags", C.c_uint32),
        ("reserved", C.c_int32), ("gemm_min_macs", C.c_double),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("op_count_lo", C.c_uint64), ("op_count_hi", C.c_uint64),
        ("d_lo", C.c_uint64), ("d_hi", C.c_uint64),
        ("width", C.c_double), ("peak_elements", C.c_uint64),
        ("work_arena_bytes", C.c_uint64), ("persistent_bytes", C.c_uint64),
        ("leaf_bytes", C.c_uint64),
        ("num_vertices", C.c_int32), ("num_hoisted", C.c_int32),
        ("num_gemm", C.c_int32), ("num_simt", C.c_int32),
        ("launches_per_slice", C.c_int32), ("out_rank", C.c_int32),
        ("out_elements", C.c_int64),
    ]


class VertexInfo(C.Structure):
    _fields_ = [
        ("ssa", C.c_int32), ("kind", C.c_int32), ("hoisted", C.c_int32), ("rank", C.c_int32),
        ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("batch", C.c_int64),
        ("macs_lo", C.c_uint64), ("macs_hi", C.c_uint64),
    ]


# every symbol include/tnx.h declares, with its ctypes signature
SIGNATURES = {
    "tnx_last_error": (C.c_char_p, []),
    "tnx_version": (C.c_char_p, []),
    "tnx_plan_create": (C.c_int, [C.POINTER(PlanDesc), C.POINTER(C.c_void_p)]),
    "tnx_plan_destroy": (C.c_int, [C.c_void_p]),
    "tnx_bind_leaves": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_void_p]),
    "tnx_run_slices": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    "tnx_run_slice_ids": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_int64, C.c_void_p]),
    "tnx_reset_accumulator": (C.c_int, [C.c_void_p, C.c_void_p]),
    "tnx_partial_result": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_void_p]),
    "tnx_partial_result_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "tnx_partial_result_exp": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int64,
                                         C.c_void_p]),
    "tnx_stats_get": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "tnx_vertex_info_get": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(VertexInfo)]),
    "tnx_debug_vertex": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.POINTER(C.c_float), C.c_int64,
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "tnx_synchronize": (C.c_int, [C.c_void_p]),
    "tnx_allreduce": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p)]),
    "tnx_profile_slice": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_float), C.POINTER(C.c_double), C.c_int32,
                                    C.POINTER(C.c_int32)]),
    "tnx_gemm_c64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                               C.c_int64, C.c_int32, C.c_void_p]),
    "tnx_clock_stamp": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "tnx_mma_peak": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.POINTER(C.c_double),
                               C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

_lib = None


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libtnx error {code}: {msg}")
        self.code = code


def load():
    """Load libtnx.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: build it with "
                           "`python -m paper_2002_01935_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc != TNX_OK:
        msg = load().tnx_last_error().decode(errors="replace")
        if rc in (TNX_ERR_INVALID, TNX_ERR_STATE):
            raise ValueError(msg)
        if rc == TNX_ERR_DATA:
            from .refpkg import DataError
            raise DataError(msg)
        if rc == TNX_ERR_NUMERIC:
            raise FloatingPointError(msg)
        if rc == TNX_ERR_OOM:
            raise MemoryError(msg)
        raise NativeError(rc, msg)


def mma_peak(kind="tf32", cta_group=2, iters=200000, stream=None):
    """Tensor-pipe ceiling measured by ``tnx_mma_peak``: (TFLOP/s, SM MHz, ms)."""
    lib = load()
    t, m, ms = C.c_double(), C.c_double(), C.c_double()
    check(lib.tnx_mma_peak({"tf32": 0, "bf16": 1, "ffma": 2}[kind], cta_group, iters, stream, C.byref(t), C.byref(m),
                           C.byref(ms)))
    return t.value, m.value, ms.value


class ClockStamps:
    """Mean SM clock over a region of a stream: ``start(stream)`` ...
    ``stop(stream)``, then ``mhz()`` after the stream has synchronised.  Each
    stamp launches ``blocks`` one-warp blocks recording (SM id, clock64,
    globaltimer); SMs seen in both stamps give cycles / ns."""

    def __init__(self, blocks=592):
        import torch
        self.blocks = blocks
        self.buf = torch.zeros((2, 3 * blocks), dtype=torch.int64, device="cuda")

    def _stamp(self, i, stream):
        check(load().tnx_clock_stamp(self.buf[i].data_ptr(), self.blocks, stream))

    def start(self, stream):
        self._stamp(0, stream)

    def stop(self, stream):
        self._stamp(1, stream)

    def mhz(self):
        a = self.buf.cpu().numpy().reshape(2, self.blocks, 3)
        first = {int(r[0]): (int(r[1]), int(r[2])) for r in a[0]}
        last = {int(r[0]): (int(r[1]), int(r[2])) for r in a[1]}
        rates = [(last[k][0] - first[k][0]) / (last[k][1] - first[k][1]) * 1e3
                 for k in first if k in last and last[k][1] > first[k][1]]
        rates.sort()
        return rates[len(rates) // 2] if rates else None, len(rates)
