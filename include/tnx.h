/*
 * tnx.h -- C ABI of the B200 sliced contraction-tree executor (libtnx.so).
 *
 * The reference (arXiv 2002.01935, package `hypertn`) is pure Python and has
 * no FFI; its hot-path entry points are the SPEC executor signatures
 *
 *   contract(tn, tree, options{strip_exponent})
 *   contract_sliced(tn, tree, slice_set, options)
 *
 * built from ContractionTree (pkg/src/hypertn/tree.py:32), annotate_incidence
 * (tree.py:137), pairwise_contract (dense.py:61) and fix_index (dense.py:161).
 * This header is the native boundary those Python signatures bind to
 * (paper_2002_01935_b200/_native.py; the ctypes stub a maintainer would add
 * on the reference side is in INTEGRATION.md).  Everything crossing it is a
 * plain pointer + size; no exceptions cross it: every call returns a
 * tnx_status and tnx_last_error() gives the thread-local message.
 *
 * Ownership: the caller owns leaf data (host or device pointers, complex128
 * or complex64, row-major in the leaf's label order); the library owns the
 * plan, its HBM arenas, CUDA graph and device accumulator.  One plan drives
 * one device; plans for different devices may be used concurrently from
 * different host threads; calls on one plan must be serialised.
 */
#ifndef TNX_H_
#define TNX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TNX_OK = 0,
  TNX_ERR_INVALID = 1,   /* ValueError in the reference (tree.py:43-56, dense.py:73/166) */
  TNX_ERR_DATA = 2,      /* DataError (network.py:18-19) */
  TNX_ERR_CUDA = 3,      /* CUDA runtime / driver failure */
  TNX_ERR_OOM = 4,       /* arena does not fit the device */
  TNX_ERR_NUMERIC = 5,   /* non-finite intermediate */
  TNX_ERR_STATE = 6      /* call out of order (e.g. run before bind) */
} tnx_status;

typedef enum {
  TNX_PREC_FP32 = 0,     /* every contraction on FP32 SIMT kernels */
  TNX_PREC_3XTF32 = 1,   /* GEMM-shaped contractions on tcgen05 tensor cores,
                            split-TF32 (hi*hi + hi*lo + lo*hi, hi and lo rounded
                            to nearest), 4M complex, FP32 accumulation in TMEM
                            promoted every 3 k-blocks with round-toward-zero
                            compensation; the rest FP32 SIMT */
  TNX_PREC_TF32_BF16X = 2 /* as 3XTF32 but the two small cross terms hi*lo +
                            lo*hi run as BF16 MMAs (2x tensor rate, ~2^-20
                            relative per product) */
} tnx_precision;

/* Leaf data element type / location for tnx_bind_leaves. */
enum { TNX_DTYPE_C128 = 0, TNX_DTYPE_C64 = 1 };
enum { TNX_LOC_HOST = 0, TNX_LOC_DEVICE = 1 };

/* Plan flags. */
enum {
  TNX_FLAG_NO_GRAPH = 1u << 0,   /* launch per-slice steps directly (debug) */
  TNX_FLAG_NO_HOIST = 1u << 1,   /* recompute slice-invariant subtrees per slice */
  TNX_FLAG_NO_TILED_PACK = 1u << 2, /* GEMM operands via the gather pack kernel only */
  TNX_FLAG_NO_DIRECT = 1u << 3,     /* no GEMM->GEMM operand-plane fusion (every
                                       intermediate materialised; debug dumps) */
  TNX_FLAG_STRIP_EXPONENT = 1u << 4 /* every intermediate rescaled to unit
                                       max-abs (exact powers of two), exponents
                                       tracked on device; read with
                                       tnx_partial_result_exp */
};

/*
 * Network + tree + slice set, interned.  Labels are integer ids 0..L-1 in the
 * reference's interning order (tn.index_table order, hypergraph.py:41-43).
 * Leaves are listed in SSA leaf order: leaf i is network node tree.leaves[i]
 * (tree.py:37-57).  pairs holds the n-1 SSA merges (a_k, b_k), merge k
 * creating vertex n+k.  sliced_labels is the SliceSet label order; slice id
 * s enumerates its assignments mixed-radix, last label fastest.
 */
typedef struct {
  int32_t num_labels;
  const int64_t* label_dims;        /* [num_labels] */
  int32_t num_leaves;
  const int32_t* leaf_ranks;        /* [num_leaves] */
  const int32_t* leaf_labels;       /* concatenated, sum(leaf_ranks) */
  const int32_t* pairs;             /* [2*(num_leaves-1)] */
  int32_t num_output;
  const int32_t* output_labels;     /* tn.output order */
  int32_t num_sliced;
  const int32_t* sliced_labels;
  int32_t precision;                /* tnx_precision */
  int32_t device;                   /* CUDA ordinal */
  uint32_t flags;
  int32_t reserved;
  double gemm_min_macs;             /* 0 -> library default */
} tnx_plan_desc;

typedef struct {
  uint64_t op_count_lo, op_count_hi;   /* per-slice MACs  sum_v U_v (128-bit) */
  uint64_t d_lo, d_hi;                 /* d_sliced (128-bit) */
  double width;                        /* W_s = log2 max internal size */
  uint64_t peak_elements;              /* 2^W_s */
  uint64_t work_arena_bytes;
  uint64_t persistent_bytes;
  uint64_t leaf_bytes;
  int32_t num_vertices;                /* internal vertices */
  int32_t num_hoisted;                 /* slice-invariant internal vertices */
  int32_t num_gemm;                    /* per-slice vertices on tcgen05 */
  int32_t num_simt;                    /* per-slice vertices on SIMT kernels */
  int32_t launches_per_slice;          /* kernels launched per slice */
  int32_t out_rank;
  int64_t out_elements;
} tnx_stats;

/* Per internal vertex description (introspection / tests). */
typedef struct {
  int32_t ssa;               /* vertex id n+k */
  int32_t kind;              /* 0 SIMT thread/out, 1 SIMT warp/out, 2 SIMT split, 3 GEMM,
                                4 full contraction (permute + streaming dot) */
  int32_t hoisted;           /* computed once per bind */
  int32_t rank;              /* rank of the result */
  int64_t m, n, k, batch;    /* GEMM-view extents */
  uint64_t macs_lo, macs_hi; /* U_v */
} tnx_vertex_info;

const char* tnx_last_error(void);
const char* tnx_version(void);

/* Compile bookkeeping, kernel choice and the HBM arena plan.  No device
 * memory is touched until tnx_bind_leaves.  */
int tnx_plan_create(const tnx_plan_desc* desc, void** plan_out);
int tnx_plan_destroy(void* plan);

/* Upload the leaves (one pointer per SSA leaf), allocate the arenas, compute
 * the slice-invariant subtrees once, capture the per-slice CUDA graph and
 * zero the accumulator.  stream may be NULL (library stream). */
int tnx_bind_leaves(void* plan, const void* const* leaf_data, int32_t dtype,
                    int32_t location, void* stream);

/* Contract slices [s_begin, s_end) and add them (compensated, complex128)
 * into the device accumulator.  Asynchronous on `stream`. */
int tnx_run_slices(void* plan, uint64_t s_begin, uint64_t s_end, void* stream);

/* Contract the slices ids[0..n) (any order, repeats allowed; each < d) and
 * add them into the accumulator, like tnx_run_slices over each id; runs of
 * consecutive ids replay the per-slice graph back to back.  The id-list form
 * of SPEC contract_sliced(..., slice_ids) and of sampled-slice runs. */
int tnx_run_slice_ids(void* plan, const uint64_t* ids, int64_t n, void* stream);

int tnx_reset_accumulator(void* plan, void* stream);

/* Copy the accumulator (complex128 interleaved, tn.output order) to host;
 * synchronises `stream`.  out_elems must equal stats.out_elements. */
int tnx_partial_result(void* plan, double* out, int64_t out_elems, void* stream);

/* As tnx_partial_result but asynchronous: the copy is enqueued on `stream`
 * and the call returns; `out` (pinned host memory for a true async copy)
 * holds the result once the stream has been synchronised.  Lets a caller
 * pipeline bind -> run -> read over many steps without a host sync each. */
int tnx_partial_result_async(void* plan, double* out, int64_t out_elems, void* stream);

/* strip_exponent plans: per output element value = out * 2^exp2. */
int tnx_partial_result_exp(void* plan, double* out, int64_t* exp2, int64_t out_elems, void* stream);

/* Single-process multi-device sum of the sliced partials (SURVEY.md §8(b)
 * "tnx_allreduce(handles[], ndev)"; the reduction the reference's SPEC
 * leaves to the caller, compensated per SPEC.md:551): every
 * plan's accumulator is replaced by the sum over all `nplans` plans (Kahan sum
 * of acc - comp in plan order, or exponent-aligned in strip_exponent mode).
 * Plans may live on different devices (peer copies over NVLink, staged by the
 * driver when peer access is off) or on the same one, must be bound and have
 * the same output size and mode.  streams[i] (or NULL / streams == NULL for
 * the library streams) orders the exchange after each plan's pending slices;
 * returns after the exchange is enqueued (tnx_partial_result synchronises).
 * Multi-process jobs (one process per GPU) use torch.distributed / NCCL over
 * tnx_partial_result instead (paper_2002_01935_b200/distributed.py). */
int tnx_allreduce(void* const* plans, int32_t nplans, void* const* streams);

int tnx_stats_get(void* plan, tnx_stats* out);
int tnx_vertex_info_get(void* plan, int32_t index, tnx_vertex_info* out);

/* Debug/parity: run slice s up to and including SSA vertex v (which must be
 * slice-dependent or hoisted) and copy its complex64 result to host together
 * with its memory layout (label ids, row-major).  */
int tnx_debug_vertex(void* plan, uint64_t s, int32_t v, float* out_c64,
                     int64_t out_elems, int32_t* layout_labels, int32_t* rank_out);

/* Profiling: run slice s (not accumulated) launch by launch on the plan's
 * stream with CUDA events around every kernel; fills up to max_launches
 * entries (type: 0 gather, 1 simt, 2 pack, 3 gemm, 4 accum; vertex = SSA id
 * or -1; ms = event-timed duration; alg_bytes = algorithmic HBM bytes of
 * memory-bound launches (permute/pack: 8 B read + 16 B written per element,
 * dot: 16 B per element), 0 for compute-bound ones) and returns the count. */
int tnx_profile_slice(void* plan, uint64_t s, int32_t* types, int32_t* vertices, float* ms,
                      double* alg_bytes, int32_t max_launches, int32_t* count);

/* Synchronise the plan's device; returns a CUDA error if one is pending. */
int tnx_synchronize(void* plan);

/* Standalone kernels exposed for unit tests / micro-benchmarks (device
 * pointers).  C[b,m,n] = sum_k A[b,m,k] B[b,n,k] over complex64 with the
 * tcgen05 split-TF32 path (A, B row-major, K innermost). */
int tnx_gemm_c64(const void* A, const void* B, void* C, int64_t batch, int64_t M,
                 int64_t N, int64_t K, int32_t precision, void* stream);

/* Tensor-pipe ceiling (diagnostic; the denominator of the GEMM roofline):
 * an MMA-only loop of `iters` tcgen05.mma (N=256; M=128 per CTA, or M=256
 * per CTA pair with cta_group 2) over shared-memory-resident pseudo-random
 * operands, one CTA per SM, no TMA / promotion / epilogue.  kind 0 =
 * kind::tf32 (K=8), 1 = kind::f16 with BF16 operands (K=16).  Returns dense
 * TFLOP/s over the device (2*M*N*K per MMA), the median SM clock the CTAs
 * measured (clock64 / globaltimer) and the event-timed duration.  kind 2 is
 * the FP32 SIMT ceiling instead: 8 independent FFMA chains per thread,
 * 4 x 256 threads per SM (cta_group ignored; 16 flop per thread-iteration). */
int tnx_mma_peak(int32_t kind, int32_t cta_group, int64_t iters, void* stream, double* tflops,
                 double* sm_mhz, double* ms);

/* Measurement: `blocks` one-warp blocks each write (SM id, clock64,
 * globaltimer ns) to device_out[3*b .. 3*b+2] on `stream`.  Two stamps around
 * a timed region give, per SM, cycles / ns = the mean SM clock over the region
 * (used by bench.py to price the roofline at the clock the kernels ran at). */
int tnx_clock_stamp(uint64_t* device_out, int32_t blocks, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TNX_H_ */
