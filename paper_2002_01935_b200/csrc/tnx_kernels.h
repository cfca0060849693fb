// Internal interface between the plan/runtime (tnx_api.cpp) and the CUDA
// kernels (kernels.cu, gemm_tc.cu).  Plain structs passed by value as kernel
// parameters; all offsets are in elements.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#ifdef __CUDACC__
// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialisation so its launch and prologue overlap the predecessor's
// tail, and waits (griddepcontrol.wait) before reading anything a predecessor
// wrote.  TNX_PDL=0 launches plainly (the wait is then a no-op).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline int pdl_enabled() {
  static const int v = getenv("TNX_PDL") ? atoi(getenv("TNX_PDL")) : 1;
  return v;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#endif

#ifdef __CUDACC__
#include <cuda_bf16.h>
#endif

namespace tnx {

constexpr int kMaxGroups = 32;   // fused label groups per index map

// Mixed-radix index map: linear index (row-major over the groups, last
// fastest) -> two operand offsets.  lg[i] >= 0 marks a power-of-two extent.
struct IdxMap {
  int32_t n;
  int32_t pad;
  int64_t dim[kMaxGroups];
  int64_t st0[kMaxGroups];
  int64_t st1[kMaxGroups];
  int8_t lg[kMaxGroups];
};

struct Int2Off { int32_t x, y; };

enum SimtMode : int32_t { SIMT_THREAD = 0, SIMT_WARP = 1, SIMT_SPLIT = 2 };

struct SimtParams {
  IdxMap out;             // output index -> (x offset, y offset)
  IdxMap sum;             // summed index -> (x offset, y offset)
  const float2* x;
  const float2* y;
  float2* z;
  float2* partial;        // SPLIT: [out_size][nsplit]
  const Int2Off* sum_tab; // optional precomputed sum offsets (int32)
  int64_t out_size;
  int64_t sum_size;
  int64_t chunk;          // SPLIT: sum elements per block
  int32_t nsplit;
  int32_t mode;
  int32_t group_lg;       // batched THREAD/WARP: 2^group_lg lanes per output (0 thread ... 5 warp)
  int32_t znp;            // > 0: the result is written as znp split-TF32 operand planes of the
                          // parent GEMM (4, or 6 for a stacked-B operand) instead of z
  float* zplanes;         // plane 0 of the parent's operand (stride zps floats per plane)
  int64_t zps;
  IdxMap zmap;            // output index -> offset in a plane (st0)
};

// Pack a complex64 tensor into fp32 planes [re_hi, re_lo, im_hi, im_lo]
// (+ [-im_hi, -im_lo] when nplanes == 6, the GEMM B operand), each
// [rows][kp] (rows = batch*R, K padded to kp with zeros); hi = x rounded to
// nearest TF32, lo = (x - hi) rounded to nearest TF32.
struct PackParams {
  IdxMap row;             // row index -> src offset (st0)
  IdxMap col;             // k index (k < K) -> src offset (st0)
  const float2* src;
  float* dst;
  int64_t rows;
  int64_t K;
  int64_t kp;
  int64_t plane_stride;   // rows * kp
  int32_t nplanes;        // 4
  int32_t mix;            // 0 split-TF32 planes, 1 mixed A-side, 2 mixed B-side
};

// Shared-memory tiled permutation (K2).  The tile spans the innermost source
// labels (coalesced reads) and the innermost destination labels (coalesced
// writes); `tab` holds three int32 tables of length ts: source offsets and
// smem slots in source iteration order, destination offsets in destination
// order.  `group` outer indices are processed per tile pass.
struct PermParams {
  IdxMap outer;           // outer index -> (src base st0, dst base st1)
  const int32_t* tab;     // [3][ts]
  const float2* src;
  void* dst;              // float planes (mode 1) or float2 (mode 0)
  int64_t n_outer;
  int64_t plane_stride;   // mode 1: elements per plane
  int32_t ts;
  int32_t group;
  int32_t mode;           // 0: complex64 copy, 1: 4 split-TF32 planes, 2: 6 planes (stacked B),
                          // 3 / 4: mixed TF32/BF16 planes for an A / B operand,
                          // 5: fused dot -- sum_i src_perm[i] * dotx[i] into per-block partials
  int32_t vec;            // 1: element pairs contiguous + aligned on both sides
  int32_t ts_log2;        // log2(ts) if ts is a power of two, else -1
  int32_t pad;
  const float2* dotx;     // mode 5: the other operand, in the destination layout
  float2* partial;        // mode 5: [gridDim.x] block partials
};

// Full contraction of two tensors in the same layout: z = sum_i x[i] y[i]
// (block partials in FP32, finalised in FP64).
struct DotParams {
  const float2* x;
  const float2* y;
  float2* z;
  float2* partial;
  int64_t n;
  int32_t nblocks;
  int32_t perm;           // >= 0: y is read through this permute (fused perm-dot), else same layout
};

constexpr int kMaxLeafRank = 16;
struct GatherJob {
  int64_t src;            // element offset in the leaf pool
  float2* dst;
  int64_t out_size;
  int32_t n_kept;
  int32_t n_sl;
  int32_t vec;            // 1: inner run contiguous, even length, every base even (16 B copies)
  int32_t pad;
  int64_t kdim[kMaxLeafRank];
  int64_t kst[kMaxLeafRank];
  uint64_t radix[kMaxLeafRank];   // suffix product of the slice dims
  int64_t sdim[kMaxLeafRank];
  int64_t sst[kMaxLeafRank];
};

// strip_exponent: per-vertex abs-max + exact power-of-two
// rescale; base-2 exponents accumulate in a device counter.
cudaError_t launch_absmax(const float2* z, int64_t n, unsigned int* bits, cudaStream_t st);
cudaError_t launch_rescale(float2* z, int64_t n, const unsigned int* bits, long long* exp_acc,
                           cudaStream_t st);

struct AccumParams {
  IdxMap out;             // output index -> root offset (st0)
  IdxMap extra;           // extra summed labels (single-leaf tree) -> root offset
  const float2* root;
  double2* acc;
  double2* comp;
  int64_t out_size;
  int64_t extra_size;
  unsigned long long* slice_counter;  // advanced by one after the slice
  // strip_exponent mode: value * 2^(hoist_exp + slice_exp) accumulated as
  // (acc, acc_exp) per element (no Kahan in this mode)
  const long long* hoist_exp;
  const long long* slice_exp;
  long long* acc_exp;
};

#ifdef __CUDACC__
// Mixed TF32/BF16 operand planes: plane words are laid out like the split-TF32
// planes ([kp/16][rows][16] 4-byte words); the bf16 "x" plane stores, per
// 16-wide k-block row, 32 bf16 = [hi(16) | lo(16)] for the A operand and
// [lo(16) | hi(16)] for B, so one bf16 MMA chunk pairs A.hi with B.lo and the
// next A.lo with B.hi (the two cross terms of the split product).
// Split-TF32 operands: hi = v rounded to nearest TF32, lo = (v - hi) rounded to
// nearest TF32.  Round-to-nearest on both parts keeps the split unbiased: the
// dropped lo*lo term and the residual v - hi - lo (<= 2^-22 |v|) carry random
// signs.  (Truncation -- masking the low 13 bits -- would make lo share the
// sign of v, so every dropped term would shrink |product| by ~1e-7 and the
// shrink would compound multiplicatively along the tree's GEMM chain.  The
// tensor core reads only the TF32 bits of each operand, so lo must itself be a
// TF32 value.)
__device__ __forceinline__ float tf32_rn(float v) {
  uint32_t r;
  asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
__device__ __forceinline__ float tf32_hi(float v) { return tf32_rn(v); }
__device__ __forceinline__ float tf32_lo(float v, float hi) { return tf32_rn(v - hi); }
__device__ __forceinline__ void store_mix_x(float* plane_x, int64_t e, float v, int side_b) {
  const float hi = tf32_hi(v);
  const float lo = v - hi;
  unsigned short* hw = reinterpret_cast<unsigned short*>(plane_x);
  const int64_t ki = e & 15;
  const int64_t base = 2 * (e - ki);
  const unsigned short hb = __bfloat16_as_ushort(__float2bfloat16_rn(hi));
  const unsigned short lb = __bfloat16_as_ushort(__float2bfloat16_rn(lo));
  hw[base + (side_b ? 16 : 0) + ki] = hb;
  hw[base + (side_b ? 0 : 16) + ki] = lb;
}
#endif

// launchers (return cudaError_t)
cudaError_t launch_gather(const GatherJob* jobs, const int32_t* block_start, int njobs,
                          int total_blocks, const float2* leaf_pool,
                          const unsigned long long* slice_counter, cudaStream_t st);
cudaError_t launch_simt(const SimtParams& p, cudaStream_t st);
// One launch for many independent thread/warp-mode SIMT contractions (one
// dependency level of the tree): block b runs job j with
// block_start[j] <= b < block_start[j+1].
cudaError_t launch_simt_batch(const SimtParams* jobs, const int32_t* block_start, int njobs,
                              int total_blocks, cudaStream_t st);
int simt_blocks(const SimtParams& p);
cudaError_t launch_pack(const PackParams& p, cudaStream_t st);
cudaError_t launch_perm(const PermParams& p, cudaStream_t st);
// fused permute + dot (mode 5): z[0] = sum over the permuted src times dotx
cudaError_t launch_perm_dot(PermParams p, float2* partial, float2* z, cudaStream_t st);
cudaError_t launch_dot(const DotParams& p, cudaStream_t st);
cudaError_t launch_accum(const AccumParams& p, cudaStream_t st);
cudaError_t launch_allreduce(const double2* acc, const double2* comp, const long long* exps, int n,
                             int64_t out_size, double2* out_acc, double2* out_comp, long long* out_exp,
                             cudaStream_t st);
cudaError_t launch_set_counter(unsigned long long* counter, unsigned long long v, cudaStream_t st);
cudaError_t launch_convert_c128(const double2* src, float2* dst, int64_t n, cudaStream_t st);
cudaError_t launch_zero(void* p, int64_t bytes, cudaStream_t st);
cudaError_t launch_clock_stamp(unsigned long long* out, int blocks, cudaStream_t st);

// tcgen05 split-TF32 complex GEMM over packed planes.
struct GemmPlan {
  alignas(64) unsigned char tmap_a[128];   // CUtensorMap
  alignas(64) unsigned char tmap_b[128];
  float2* out;
  int64_t M, N, kp, batch;
  int32_t ok;
  int32_t promote;        // k-blocks (of 16) per TMEM accumulation round
  int32_t splits;         // split-K factor (1 = none)
  int32_t two_sm;         // 2-CTA (cta_group::2) variant
  float2* partial;        // split-K workspace [splits][batch][M][N]
  // direct planes: write the result as the parent GEMM's split-TF32 operand
  // planes (offset = fmap(row) + gmap(col)) instead of complex64 `out`
  int32_t direct;
  int32_t dvec;           // direct stores as float4 runs of 4 columns
  int32_t mix;            // mixed TF32/BF16 mode (operand planes and MMA sequence)
  int32_t dmix;           // direct planes in the mixed format for parent side dside
  int32_t dside;
  int32_t stackb;         // stacked-B 2-CTA variant: B planes carry -im_hi, -im_lo (6 planes)
  int32_t dstack;         // direct planes of a stacked-B parent's B operand (write 6 planes)
  int32_t dpair;          // direct planes: 16 consecutive rows are 64 contiguous bytes and column
                          // pairs adjacent 64 B chunks -> full-line stores (epilogue exchanges lanes)
  float* dplanes;
  int64_t dplane_stride;
  IdxMap fmap;            // output row (batch*M + m) -> plane offset (st0)
  IdxMap gmap;            // output column n -> plane offset (st0)
};
// Build tensor maps for planes laid out as [4][batch][M|N][kp] fp32; kp a
// multiple of 16.
int gemm_prepare(GemmPlan* g, const float* a_planes, const float* b_planes, float2* out,
                 int64_t batch, int64_t M, int64_t N, int64_t kp, int splits, float2* partial,
                 char* err, size_t errlen, int stack_b = 0);
int gemm_choose_splits(int64_t batch, int64_t M, int64_t N, int64_t kp);
int gemm_use_2sm(int64_t batch, int64_t M, int64_t N, int64_t kp, int splits);
// stacked-B 2-CTA variant enabled (TNX_GEMM_STACKB=0 disables)
int gemm_stack_enabled();
// stacked B for this shape (cost model; requires the 2-CTA configuration)
int gemm_use_stack(int64_t batch, int64_t M, int64_t N, int64_t kp, int two_sm);
cudaError_t launch_gemm(const GemmPlan& g, cudaStream_t st);
int gemm_init_attributes(char* err, size_t errlen);
// MMA-only tensor-pipe ceiling (no TMA / epilogue; kind 0 tf32, 1 bf16) or the
// FP32 FFMA ceiling (kind 2): TFLOP/s, median SM MHz
int gemm_mma_peak(int kind, int two_sm, int64_t iters, cudaStream_t st, double* tflops, double* sm_mhz,
                  double* ms, char* err, size_t errlen);

}  // namespace tnx
