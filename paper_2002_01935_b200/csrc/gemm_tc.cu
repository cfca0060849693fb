// K3: tcgen05 / TMEM / TMA complex64 GEMM with split-TF32 (3 passes) and the
// 4M complex decomposition, for the GEMM-shaped pairwise contractions of the
// tree (reference pairwise_contract -> np.einsum -> zgemm, dense.py:47-76).
//
//   C[b,m,n] = sum_k A[b,m,k] * B[b,n,k]          (complex64 in/out)
//
//   Cre += Ar_h Br_h + Ar_h Br_l + Ar_l Br_h - (Ai_h Bi_h + Ai_h Bi_l + Ai_l Bi_h)
//   Cim += Ar_h Bi_h + Ar_h Bi_l + Ar_l Bi_h +  Ai_h Br_h + Ai_h Br_l + Ai_l Br_h
//
// Operands are fp32 planes [re_hi, re_lo, im_hi, im_lo] (+ [-im_hi, -im_lo]
// for a stacked-B operand), K-blocked [plane][kp/16][batch*rows][16] so every
// TMA box (3-D tensor map) is one contiguous block; written by the pack /
// permute kernels or directly by a child GEMM's epilogue.
//
// One persistent kernel template, instantiated per (2-CTA pair, precision,
// epilogue mode, stacked B): warp 0 lane 0 = TMA producer (smem ring), warp 1
// lane 0 = MMA issuer, warps 2-9 = promotion + epilogue.
//   * 1-CTA: 128x128 tiles, 12 tcgen05.mma (N=128) per 8-wide k-step.
//   * 2-CTA (cta_group::2): 256x128 pair tiles, each CTA stages its 128 A rows
//     and half of B.  Stacked B: each CTA stages full 128-row B slots
//     ([re|-im] / [im|re]) and 6 N=256 MMAs per k-step accumulate straight into
//     the [Re | Im] TMEM columns (shared-memory operand traffic -17 %).
//   * Tensor-core accumulation rounds toward zero, so every `promote` k-blocks
//     (the first round of a unit: `first`) the TMEM accumulator set (two sets,
//     double-buffered) is added into FP32 registers of the epilogue warps,
//     which release it with a relaxed mbarrier arrive.
//   * Epilogue: interleaved complex64, split-K partials, or the parent GEMM's
//     operand planes (GEMM->GEMM fusion).
//   * Launch: cost model over (2-CTA, split-K), grid = min(units, SMs / pairs),
//     programmatic dependent launch (griddepcontrol.wait after the prologue).
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tnx_kernels.h"

namespace tnx {

namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 16;                          // fp32 per smem row (64 B, SWIZZLE_64B)
constexpr int TMEM_COLS = 512;
constexpr int GROUP_M = 8;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t mbar, int c0,
                                            int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(mbar), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}

// L2 policy of the operand loads: evict_last (operands are re-read by the other
// tiles of the wave) or evict_normal (TNX_GEMM_L2HINT=0)
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t p;
  if (keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_64B, rows of 64 B,
// 8-row groups 512 B apart (SBO), LBO unused (=1), sm100 version bit.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(512u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)4u << 61;
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// kind::f16 with BF16 operands (cross terms of the mixed TF32/BF16 mode)
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct GemmArgs {
  float2* out;
  int64_t M, N, batch;
  int32_t num_kb;        // kp / BK
  int32_t tiles_m, tiles_n;
  int32_t promote;       // k-blocks accumulated in TMEM before promotion
  int32_t group_m;       // rasterisation: M tiles per group
  int32_t kb_per_split;  // split-K: k-blocks per work unit
  int32_t splits;        // split-K slices (work units per tile)
  float2* partial;       // split-K workspace [splits][batch][M][N] (nullptr: 1 split)
  int64_t rows_a, rows_b;  // batch * M, batch * N (rows per plane)
  int32_t direct;        // 1: store as the parent's split-TF32 planes
  int32_t dvec;          // direct stores in float4 runs
  int32_t mix;           // 1: TF32 hi*hi + BF16 cross terms (planes re_hi, re_x, im_hi, im_x)
  int32_t dmix;          // direct planes in the mixed format ...
  int32_t dside;         // ... for the parent's A (0) or B (1) operand
  float* dplanes;
  int64_t dplane_stride;
  IdxMap fmap, gmap;
  int32_t debug;         // TNX_GEMM_DEBUG bit 0: skip the TMA loads, bit 1: skip the epilogue stores,
                         // bit 2 / 3: paired direct planes without the negated planes / plane 0 only,
                         // bit 5: no MMAs (pipeline ceilings; wrong results)
  int32_t dstack;        // direct planes of a stacked-B parent operand: also write -im_hi, -im_lo (planes 4, 5)
  int32_t dpair;         // direct planes in full-line pairs (see epilogue_store)
  int32_t ksnake;        // odd waves traverse K in reverse (L2 reuse across waves)
  int32_t first;         // k-blocks of a unit's first TMEM round (>= promote; see launch_gemm)
  float rz_kappa;        // round-toward-zero compensation (see the promotion loop); 0 disables
  int32_t l2keep;        // operand loads with an L2 evict_last policy (TNX_GEMM_L2HINT bit 0)
  int32_t stcs;          // results stored evict-first (bit 1)
};

__device__ __forceinline__ int64_t map_offset(const IdxMap& m, int64_t idx) {
  int64_t o = 0;
#pragma unroll 1
  for (int i = m.n - 1; i >= 0; --i) {
    int64_t r;
    if (m.lg[i] >= 0) {
      r = idx & (m.dim[i] - 1);
      idx >>= m.lg[i];
    } else {
      const int64_t q = idx / m.dim[i];
      r = idx - q * m.dim[i];
      idx = q;
    }
    o += r * m.st0[i];
  }
  return o;
}

// result stores: plain, or streaming (st.global.cs, evict-first) with
// TNX_GEMM_L2HINT bit 1
__device__ __forceinline__ void st_res(float4* p, float4 v, bool cs) {
  if (cs) __stcs(p, v); else *p = v;
}
__device__ __forceinline__ void st_res(float* p, float v, bool cs) {
  if (cs) __stcs(p, v); else *p = v;
}

// Epilogue store of one thread's 64 promoted columns of row `row` (global
// row index b*M + m).  Plain mode: interleaved complex64.  Direct mode: the
// four split-TF32 planes of the parent GEMM operand, column offsets from the
// per-CTA table `gtab` (built by the epilogue warps once the main loop is
// done and the pipeline's shared memory is free).
// EPI: 0 interleaved complex64 (or split-K partials), 1 direct planes (scalar
// stores), 2 direct planes in float4 runs (scalar fallback for edge tiles).
// Templated so each kernel instance carries only its own store code.
// EPI 0 stages through shared memory (`stg`, 32 rows x 80 B per warp): a warp's
// 32 lanes hold 32 rows, so direct row stores would touch 32 lines per
// instruction (ncu: LSU throttling, and the MMA then waited for the epilogue on
// mid-K GEMMs); transposed 8 columns at a time, each store instruction writes
// 8 rows x 64 contiguous bytes.
template <int EPI, bool MIX>
__device__ __forceinline__ void epilogue_store(const GemmArgs& g, float2* out, int64_t grow,
                                               bool row_ok, int64_t col0, int hcol,
                                               const float (&mre)[64], const float (&mim)[64],
                                               const int64_t* gtab, unsigned char* stg) {
  if constexpr (EPI == 0) {
    if (col0 + 64 <= g.N && (g.N & 1) == 0 && __all_sync(0xffffffffu, row_ok)) {
      const int lane = threadIdx.x & 31;
      const int64_t grow0 = grow - lane;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        float4* w = reinterpret_cast<float4*>(stg + lane * 80);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          w[k] = make_float4(mre[8 * c + 2 * k], mim[8 * c + 2 * k], mre[8 * c + 2 * k + 1],
                             mim[8 * c + 2 * k + 1]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = i * 8 + (lane >> 2), q = lane & 3;
          const float4 v = *reinterpret_cast<const float4*>(stg + r * 80 + q * 16);
          st_res(reinterpret_cast<float4*>(out + (grow0 + r) * g.N + col0 + 8 * c) + q, v, g.stcs);
        }
        __syncwarp();
      }
      return;
    }
  }
  // EPI 1, paired lines: when 16 consecutive rows are 64 contiguous bytes of a
  // plane and columns 2c, 2c+1 are adjacent 64 B chunks (g.dpair), lanes 0-15
  // (rows r..r+15) and 16-31 (rows r+16..r+31) swap one value per column pair
  // so each store instruction writes two whole 128 B lines -- half the store
  // requests of one 64 B segment per half-warp, and the L1->crossbar request
  // path is shared with the TMA operand loads (ncu: the mid-K GEMMs' stores
  // starved the loads).
  if constexpr (EPI == 1 && !MIX) {
    if (g.dpair && col0 + 64 <= g.N && __all_sync(0xffffffffu, row_ok)) {
      const int lane = threadIdx.x & 31;
      const bool up = lane >= 16;
      const int64_t f = map_offset(g.fmap, grow);
      const int64_t fa = __shfl_sync(0xffffffffu, f, lane & 15);         // row (lane & 15)
      const int64_t fb = __shfl_sync(0xffffffffu, f, (lane & 15) + 16);  // row (lane & 15) + 16
      float* d = g.dplanes;
      const int64_t ps = g.dplane_stride;
      const int64_t sh = up ? 16 : 0;
#pragma unroll
      for (int j = 0; j < 64; j += 2) {
        const int64_t oj = gtab[hcol + j];
        float v[2][4];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          v[c][0] = tf32_hi(mre[j + c]);
          v[c][1] = tf32_lo(mre[j + c], v[c][0]);
          v[c][2] = tf32_hi(mim[j + c]);
          v[c][3] = tf32_lo(mim[j + c], v[c][2]);
        }
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const float recv = __shfl_xor_sync(0xffffffffu, up ? v[0][p] : v[1][p], 16);
          const float a = up ? recv : v[0][p];   // line of rows 0-15: columns j | j+1
          const float b = up ? v[1][p] : recv;   // line of rows 16-31
          if ((g.debug & 8) && p > 0) continue;  // debug: plane 0 only
          st_res(d + fa + oj + sh + p * ps, a, g.stcs);
          st_res(d + fb + oj + sh + p * ps, b, g.stcs);
          if (g.dstack && p >= 2 && !(g.debug & 4)) {  // planes 4, 5: -im_hi, -im_lo
            st_res(d + fa + oj + sh + (p + 2) * ps, -a, g.stcs);
            st_res(d + fb + oj + sh + (p + 2) * ps, -b, g.stcs);
          }
        }
      }
      return;
    }
  }
  if (!row_ok) return;
  if (EPI == 2 && col0 + 64 <= g.N) {
    const int64_t f = map_offset(g.fmap, grow);
    float* d = g.dplanes;
    const int64_t ps = g.dplane_stride;
#pragma unroll
    for (int j = 0; j < 64; j += 4) {
      const int64_t off = f + gtab[hcol + j];
      if constexpr (MIX) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          d[off + t] = tf32_hi(mre[j + t]);
          d[off + 2 * ps + t] = tf32_hi(mim[j + t]);
          store_mix_x(d + ps, off + t, mre[j + t], g.dside);
          store_mix_x(d + 3 * ps, off + t, mim[j + t], g.dside);
        }
      } else {
        float rh[4], rl[4], ih[4], il[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          rh[t] = tf32_hi(mre[j + t]);
          ih[t] = tf32_hi(mim[j + t]);
          rl[t] = tf32_lo(mre[j + t], rh[t]);
          il[t] = tf32_lo(mim[j + t], ih[t]);
        }
        st_res(reinterpret_cast<float4*>(d + off), make_float4(rh[0], rh[1], rh[2], rh[3]), g.stcs);
        st_res(reinterpret_cast<float4*>(d + off + ps), make_float4(rl[0], rl[1], rl[2], rl[3]), g.stcs);
        st_res(reinterpret_cast<float4*>(d + off + 2 * ps), make_float4(ih[0], ih[1], ih[2], ih[3]), g.stcs);
        st_res(reinterpret_cast<float4*>(d + off + 3 * ps), make_float4(il[0], il[1], il[2], il[3]), g.stcs);
        if (g.dstack) {
          st_res(reinterpret_cast<float4*>(d + off + 4 * ps), make_float4(-ih[0], -ih[1], -ih[2], -ih[3]), g.stcs);
          st_res(reinterpret_cast<float4*>(d + off + 5 * ps), make_float4(-il[0], -il[1], -il[2], -il[3]), g.stcs);
        }
      }
    }
    return;
  }
  if constexpr (EPI >= 1) {
    const int64_t f = map_offset(g.fmap, grow);
    float* d = g.dplanes;
    const int64_t ps = g.dplane_stride;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      if (col0 + j >= g.N) continue;
      const int64_t off = f + gtab[hcol + j];
      const float re = mre[j], im = mim[j];
      const float rh = tf32_hi(re);
      const float ih = tf32_hi(im);
      st_res(d + off, rh, g.stcs);
      st_res(d + off + 2 * ps, ih, g.stcs);
      if constexpr (MIX) {
        store_mix_x(d + ps, off, re, g.dside);
        store_mix_x(d + 3 * ps, off, im, g.dside);
      } else {
        const float il = tf32_lo(im, ih);
        st_res(d + off + ps, tf32_lo(re, rh), g.stcs);
        st_res(d + off + 3 * ps, il, g.stcs);
        if (g.dstack) {
          st_res(d + off + 4 * ps, -ih, g.stcs);
          st_res(d + off + 5 * ps, -il, g.stcs);
        }
      }
    }
    return;
  }
  float2* orow = out + grow * g.N;
  if (col0 + 64 <= g.N && (g.N & 1) == 0) {
    float4* dst = reinterpret_cast<float4*>(orow + col0);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      st_res(dst + j, make_float4(mre[2 * j], mim[2 * j], mre[2 * j + 1], mim[2 * j + 1]), g.stcs);
  } else {
#pragma unroll
    for (int j = 0; j < 64; ++j)
      if (col0 + j < g.N) orow[col0 + j] = make_float2(mre[j], mim[j]);
  }
}

// TMEM-set release by the epilogue warps.  Relaxed: the MMA issuer only needs
// the promotion's TMEM reads done (tcgen05.wait::ld + tcgen05.fence::
// before_thread_sync precede the arrive); a release arrive would also make every
// thread wait for its previous tile's global stores to become visible
// (MEMBAR.GPU), serialising the epilogue stores with the next tile's MMAs.
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

// Warp roles: 0 = TMA producer, 1 = MMA issuer, 2..9 = promotion/epilogue.
// Tensor-core accumulation rounds toward zero, so its error grows with the
// number of MMAs folded into one accumulator.  Every `promote` k-blocks the
// MMA issuer switches to the other TMEM accumulator set (double buffered,
// 2 x 256 columns) while the epilogue warps add the finished set into FP32
// registers with round-to-nearest ("promotion", as done for FP8 GEMMs).
//
// The kernel is persistent: each CTA (or CTA pair) walks work units
// (tile, batch, split-K slice) with a stride of the grid; the smem ring and
// the TMEM round counter run continuously across units, so the epilogue
// stores of one tile overlap the first MMA rounds of the next.
//
// TWO_SM: a cluster of two CTAs on one TPC computes a 256 x 128 tile with
// tcgen05.mma.cta_group::2 (M = 256) issued by the leader; each CTA stages
// its own 128 A rows and half of the B tile (64 rows) per plane, so per-SM
// shared-memory operand traffic per MMA drops from 8 KB to 6 KB.  TMA loads
// of both CTAs complete on the leader's "full" barrier (peer bit cleared),
// MMA commits multicast to both CTAs' "empty" / "tmem full" barriers, and
// both CTAs' epilogue warps release a TMEM set on the leader's barrier.
constexpr int NUM_THREADS = 320;
constexpr int BN_HALF = BN / 2;
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;

// STACK (2-CTA, 3xTF32 only): "stacked B".  Each CTA stages four full
// 128-row B slots, CTA0 {re_hi, re_lo, -im_hi, -im_lo} and CTA1 {im_hi,
// im_lo, re_hi, re_lo}, so one N=256 MMA A_re x [B_re | B_im] (slots 0/1) and
// one A_im x [-B_im | B_re] (slots 2/3) accumulate straight into the
// [Re | Im] TMEM columns: 12 MMAs of N=256 per k-block instead of 24 of N=128,
// shared-memory operand traffic per k-block 144 + 48 KB -> 96 + 64 KB.  The B
// operand carries two extra planes (-im_hi, -im_lo; planes 4, 5).
template <bool TWO_SM, bool STACK = false>
struct KCfg {
  static constexpr int A_BYTES = BM * BK * 4;                                        // 8 KB
  static constexpr int B_BYTES = (TWO_SM && !STACK ? BN_HALF : BN) * BK * 4;         // 4 / 8 KB
  static constexpr int STAGE = 4 * A_BYTES + 4 * B_BYTES;                            // 48 / 64 KB
  static constexpr int NSTAGE = TWO_SM && !STACK ? 4 : 3;
  static constexpr int GTAB_OFF = NSTAGE * STAGE;                      // 1 KB column table
  static constexpr int BAR_OFF = GTAB_OFF + BN * 8;
  static constexpr int STG_OFF = BAR_OFF + 256;                        // EPI 0 staging: 8 warps x 2.5 KB
  static constexpr int STG_ROW = 80;                                   // 8 complex + 16 B pad (bank spread)
  static constexpr int STG_WARP = 32 * STG_ROW;
  static constexpr int SMEM = STG_OFF + 8 * STG_WARP + 1024;
  static constexpr int TILE_M = TWO_SM ? 256 : BM;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm(uint32_t dst, const void* tmap, uint32_t mbar, int c0, int c1,
                                                int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(mbar & PEER_MASK), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_tf32_2sm(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_2sm(uint32_t mbar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(mbar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint32_t local_addr) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(0));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// idesc: D=f32, A=B=tf32 (fmt 2) or bf16 (fmt 1), K-major, N=128, M=128 (1 CTA)
// or 256 (pair)
template <bool TWO_SM>
__host__ __device__ constexpr uint32_t idesc_mma(bool neg_a, uint32_t fmt = 2u, int n = BN) {
  return (1u << 4) | (fmt << 7) | (fmt << 10) | ((neg_a ? 1u : 0u) << 13) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)((TWO_SM ? 256 : BM) >> 4) << 24);
}

// work unit -> (split z, batch b, tile row tm, tile column tn)
__device__ __forceinline__ void decode_unit(const GemmArgs& g, int u, int& z, int& b, int& tm, int& tn) {
  const int tiles = g.tiles_m * g.tiles_n;
  const int t = u % tiles;
  const int zb = u / tiles;
  b = zb % (int)g.batch;
  z = zb / (int)g.batch;
  const int group_span = g.group_m * g.tiles_n;
  const int group = t / group_span;
  const int first_m = group * g.group_m;
  const int gm = min(g.tiles_m - first_m, g.group_m);
  tm = first_m + (t % group_span) % gm;
  tn = (t % group_span) / gm;
}

template <bool TWO_SM, bool MIX, int EPI, bool STACK>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_c64_3xtf32_kernel(const __grid_constant__ CUtensorMap tm_a,
                           const __grid_constant__ CUtensorMap tm_b, const GemmArgs g) {
  static_assert(!STACK || (TWO_SM && !MIX), "stacked B is a 2-CTA 3xTF32 variant");
  using C = KCfg<TWO_SM, STACK>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  int64_t* gtab = reinterpret_cast<int64_t*>(smem + C::GTAB_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::NSTAGE;
  uint64_t* tfull = bars + 2 * C::NSTAGE;
  uint64_t* tempty = bars + 2 * C::NSTAGE + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::NSTAGE + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = TWO_SM ? cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int cid = TWO_SM ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int ncta = TWO_SM ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int units = g.tiles_m * g.tiles_n * (int)g.batch * g.splits;

  if (warp == 0) {
    if constexpr (TWO_SM) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_addr(tmem_slot)), "r"(TMEM_COLS) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_addr(tmem_slot)), "r"(TMEM_COLS) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < C::NSTAGE; ++s) {
      mbar_init(smem_addr(&full[s]), 1);
      mbar_init(smem_addr(&empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_addr(&tfull[s]), 1);
      mbar_init(smem_addr(&tempty[s]), TWO_SM ? 16 : 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  if constexpr (TWO_SM) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  // prologue above (TMEM allocation, barrier init) overlaps the predecessor's
  // tail under programmatic dependent launch; its outputs are read only below
  pdl_wait();
  const uint32_t tmem_base = *tmem_slot;
  const int P = g.promote;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const uint64_t pol = l2_policy(g.l2keep != 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < units; u += ncta) {
        int z, b, tm, tn;
        decode_unit(g, u, z, b, tm, tn);
        const int kb_begin = z * g.kb_per_split;
        const int nkb = min(g.num_kb - kb_begin, g.kb_per_split);
        const int row_a = (int)(b * g.M + (int64_t)tm * C::TILE_M + rank * BM);
        const int row_b = (int)(b * g.N + (int64_t)tn * BN + (STACK ? 0 : rank * BN_HALF));
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(smem_addr(&empty[stage]), phase ^ 1u);
          const uint32_t fb = smem_addr(&full[stage]);
          if (g.debug & 1) {
            if (leader) mbar_expect_tx(fb, 0);
            if (++stage == C::NSTAGE) {
              stage = 0;
              phase ^= 1u;
            }
            continue;
          }
          if (leader) mbar_expect_tx(fb, (TWO_SM ? 2 : 1) * C::STAGE);
          unsigned char* sbase = smem + stage * C::STAGE;
          // k-snake: odd waves of the persistent grid walk K backwards, so they
          // start on the k-slices the previous wave (same A rows under group-M
          // rasterisation) left in L2
          const int kbg = kb_begin + ((g.ksnake && (((u - cid) / ncta) & 1)) ? nkb - 1 - kb : kb);
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            if constexpr (STACK) {
              // B slot p of this CTA: CTA0 planes {0, 1, 4, 5}, CTA1 {2, 3, 0, 1}
              const int bp = rank == 0 ? (p < 2 ? p : p + 2) : (p < 2 ? p + 2 : p - 2);
              tma_load_3d_2sm(smem_addr(sbase + p * C::A_BYTES), &tm_a, fb, 0, row_a, p * g.num_kb + kbg, pol);
              tma_load_3d_2sm(smem_addr(sbase + 4 * C::A_BYTES + p * C::B_BYTES), &tm_b, fb, 0, row_b,
                              bp * g.num_kb + kbg, pol);
            } else if constexpr (TWO_SM) {
              tma_load_3d_2sm(smem_addr(sbase + p * C::A_BYTES), &tm_a, fb, 0, row_a, p * g.num_kb + kbg, pol);
              tma_load_3d_2sm(smem_addr(sbase + 4 * C::A_BYTES + p * C::B_BYTES), &tm_b, fb, 0, row_b,
                              p * g.num_kb + kbg, pol);
            } else {
              tma_load_3d(smem_addr(sbase + p * C::A_BYTES), &tm_a, fb, 0, row_a, p * g.num_kb + kbg, pol);
              tma_load_3d(smem_addr(sbase + 4 * C::A_BYTES + p * C::B_BYTES), &tm_b, fb, 0, row_b,
                          p * g.num_kb + kbg, pol);
            }
          }
          if (++stage == C::NSTAGE) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t ID_POS = idesc_mma<TWO_SM>(false);
      constexpr uint32_t ID_NEG = idesc_mma<TWO_SM>(true);
      constexpr uint32_t ID_BP = idesc_mma<TWO_SM>(false, 1u);
      constexpr uint32_t ID_BN = idesc_mma<TWO_SM>(true, 1u);
      constexpr uint32_t ID_S = idesc_mma<TWO_SM>(false, 2u, 2 * BN);  // N = 256 (stacked B)
      int stage = 0;
      uint32_t phase = 0;
      uint32_t R = 0;  // global accumulator-round counter
      for (int u = cid; u < units; u += ncta) {
        int z, b, tm, tn;
        decode_unit(g, u, z, b, tm, tn);
        const int kb_begin = z * g.kb_per_split;
        const int nkb = min(g.num_kb - kb_begin, g.kb_per_split);
        const int F = min(nkb, max(P, g.first));  // first TMEM round of the unit
        const int rounds = 1 + (nkb - F + P - 1) / P;
        for (int r = 0; r < rounds; ++r, ++R) {
          const uint32_t set = R & 1u;
          mbar_wait(smem_addr(&tempty[set]), ((R >> 1) & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t d_re = tmem_base + set * 256;
          const uint32_t d_im = d_re + BN;
          const int kb0 = r == 0 ? 0 : F + (r - 1) * P;
          const int kb1 = r == 0 ? F : min(nkb, kb0 + P);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(smem_addr(&full[stage]), phase);
            tc_fence_after();
            const uint32_t sb = smem_addr(smem + stage * C::STAGE);
#pragma unroll
            for (int ks = 0; ks < BK / 8; ++ks) {
              const uint32_t koff = ks * 32;
              const uint64_t ar_h = umma_desc_sw64(sb + 0 * C::A_BYTES + koff);
              const uint64_t ar_l = umma_desc_sw64(sb + 1 * C::A_BYTES + koff);
              const uint64_t ai_h = umma_desc_sw64(sb + 2 * C::A_BYTES + koff);
              const uint64_t ai_l = umma_desc_sw64(sb + 3 * C::A_BYTES + koff);
              const uint32_t bb = sb + 4 * C::A_BYTES + koff;
              const uint64_t br_h = umma_desc_sw64(bb + 0 * C::B_BYTES);
              const uint64_t br_l = umma_desc_sw64(bb + 1 * C::B_BYTES);
              const uint64_t bi_h = umma_desc_sw64(bb + 2 * C::B_BYTES);
              const uint64_t bi_l = umma_desc_sw64(bb + 3 * C::B_BYTES);
              const uint32_t acc0 = (kb > kb0 || ks > 0) ? 1u : 0u;
              if (g.debug & 32) continue;  // debug: no MMAs (operand-streaming ceiling)
              if constexpr (STACK) {
                // slots: 0 [re_hi | im_hi], 1 [re_lo | im_lo], 2 [-im_hi | re_hi], 3 [-im_lo | re_lo]
                umma_tf32_2sm(d_re, ar_h, br_l, ID_S, acc0);  // hi.lo
                umma_tf32_2sm(d_re, ar_l, br_h, ID_S, 1u);    // lo.hi
                umma_tf32_2sm(d_re, ai_h, bi_l, ID_S, 1u);
                umma_tf32_2sm(d_re, ai_l, bi_h, ID_S, 1u);
                umma_tf32_2sm(d_re, ar_h, br_h, ID_S, 1u);    // hi.hi
                umma_tf32_2sm(d_re, ai_h, bi_h, ID_S, 1u);
                continue;
              }
              if constexpr (MIX) {
                // planes: 0 re_hi (tf32), 1 re_x (bf16 [hi|lo] / [lo|hi]), 2 im_hi, 3 im_x
                if constexpr (TWO_SM) {
                  umma_bf16_2sm(d_re, ar_l, br_l, ID_BP, acc0);
                  umma_bf16_2sm(d_re, ai_l, bi_l, ID_BN, 1u);
                  umma_tf32_2sm(d_re, ar_h, br_h, ID_POS, 1u);
                  umma_tf32_2sm(d_re, ai_h, bi_h, ID_NEG, 1u);
                  umma_bf16_2sm(d_im, ar_l, bi_l, ID_BP, acc0);
                  umma_bf16_2sm(d_im, ai_l, br_l, ID_BP, 1u);
                  umma_tf32_2sm(d_im, ar_h, bi_h, ID_POS, 1u);
                  umma_tf32_2sm(d_im, ai_h, br_h, ID_POS, 1u);
                } else {
                  umma_bf16(d_re, ar_l, br_l, ID_BP, acc0);
                  umma_bf16(d_re, ai_l, bi_l, ID_BN, 1u);
                  umma_tf32(d_re, ar_h, br_h, ID_POS, 1u);
                  umma_tf32(d_re, ai_h, bi_h, ID_NEG, 1u);
                  umma_bf16(d_im, ar_l, bi_l, ID_BP, acc0);
                  umma_bf16(d_im, ai_l, br_l, ID_BP, 1u);
                  umma_tf32(d_im, ar_h, bi_h, ID_POS, 1u);
                  umma_tf32(d_im, ai_h, br_h, ID_POS, 1u);
                }
                continue;
              }
              if constexpr (TWO_SM) {
                umma_tf32_2sm(d_re, ar_h, br_l, ID_POS, acc0);
                umma_tf32_2sm(d_re, ar_l, br_h, ID_POS, 1u);
                umma_tf32_2sm(d_re, ai_h, bi_l, ID_NEG, 1u);
                umma_tf32_2sm(d_re, ai_l, bi_h, ID_NEG, 1u);
                umma_tf32_2sm(d_re, ar_h, br_h, ID_POS, 1u);
                umma_tf32_2sm(d_re, ai_h, bi_h, ID_NEG, 1u);
                umma_tf32_2sm(d_im, ar_h, bi_l, ID_POS, acc0);
                umma_tf32_2sm(d_im, ar_l, bi_h, ID_POS, 1u);
                umma_tf32_2sm(d_im, ai_h, br_l, ID_POS, 1u);
                umma_tf32_2sm(d_im, ai_l, br_h, ID_POS, 1u);
                umma_tf32_2sm(d_im, ar_h, bi_h, ID_POS, 1u);
                umma_tf32_2sm(d_im, ai_h, br_h, ID_POS, 1u);
              } else {
                umma_tf32(d_re, ar_h, br_l, ID_POS, acc0);
                umma_tf32(d_re, ar_l, br_h, ID_POS, 1u);
                umma_tf32(d_re, ai_h, bi_l, ID_NEG, 1u);
                umma_tf32(d_re, ai_l, bi_h, ID_NEG, 1u);
                umma_tf32(d_re, ar_h, br_h, ID_POS, 1u);
                umma_tf32(d_re, ai_h, bi_h, ID_NEG, 1u);
                umma_tf32(d_im, ar_h, bi_l, ID_POS, acc0);
                umma_tf32(d_im, ar_l, bi_h, ID_POS, 1u);
                umma_tf32(d_im, ai_h, br_l, ID_POS, 1u);
                umma_tf32(d_im, ai_l, br_h, ID_POS, 1u);
                umma_tf32(d_im, ar_h, bi_h, ID_POS, 1u);
                umma_tf32(d_im, ai_h, br_h, ID_POS, 1u);
              }
            }
            if constexpr (TWO_SM) umma_commit_2sm(smem_addr(&empty[stage]));
            else umma_commit(smem_addr(&empty[stage]));
            if (++stage == C::NSTAGE) {
              stage = 0;
              phase ^= 1u;
            }
          }
          if constexpr (TWO_SM) umma_commit_2sm(smem_addr(&tfull[set]));
          else umma_commit(smem_addr(&tfull[set]));
        }
      }
    }
  } else {
    // ---------------- promotion + epilogue (8 warps per CTA) ----------------
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int h = (warp - 2) >> 2;   // column half
    const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16) + h * 64;
    uint32_t R = 0;
    for (int u = cid; u < units; u += ncta) {
      int z, b, tm, tn;
      decode_unit(g, u, z, b, tm, tn);
      const int kb_begin = z * g.kb_per_split;
      const int nkb = min(g.num_kb - kb_begin, g.kb_per_split);
      const int rounds = 1 + (nkb - min(nkb, max(P, g.first)) + P - 1) / P;
      float mre[64], mim[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        mre[j] = 0.f;
        mim[j] = 0.f;
      }
      const int F = min(nkb, max(P, g.first));
      for (int r = 0; r < rounds; ++r, ++R) {
        const uint32_t set = R & 1u;
        mbar_wait(smem_addr(&tfull[set]), (R >> 1) & 1u);
        tc_fence_after();
        const uint32_t t0 = lane_base + set * 256;
        // Round-toward-zero compensation.  The tensor core truncates the FP32
        // accumulator after every MMA, so each of the round's 12 MMAs per
        // k-block (6 per 8-wide k-step: four split cross terms, then the two
        // hi*hi terms) shrinks the partial sum S_j by 0.5 ulp(S_j) on average,
        // i.e. by E[ulp/|S|]/2 = 2^-24 / (2 ln 2) ~ 0.72 * 2^-24 relative for
        // log-uniformly distributed mantissas.  With exchangeable k-step
        // increments E[S_j | S] is linear in j, so the expected shrink of the
        // round's sum S is 2^-24 kappa (6 n_kb - 2) S (n_kb k-blocks per round;
        // the four cross-term MMAs of a k-step act on the previous k-step's
        // partial).  Promotion adds S (1 + that) -- an unbiased estimate, so the
        // residual error is the zero-mean part that grows like sqrt(n).
        const int nkb_r = r == 0 ? F : min(nkb - F - (r - 1) * P, P);
        // (mixed TF32/BF16 mode: 8 MMAs per k-block -- two BF16 cross-term MMAs,
        // then the two TF32 hi*hi ones, per k-step -- giving 4 n_kb - 1)
        const float delta = g.rz_kappa * 5.9604645e-8f * (float)(MIX ? 4 * nkb_r - 1 : 6 * nkb_r - 2);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t re[32], im[32];
          tmem_ld32(t0 + j * 32, re);
          tmem_ld32(t0 + BN + j * 32, im);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const float vr = __uint_as_float(re[t]), vi = __uint_as_float(im[t]);
            mre[j * 32 + t] = fmaf(vr, delta, mre[j * 32 + t] + vr);
            mim[j * 32 + t] = fmaf(vi, delta, mim[j * 32 + t] + vi);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (TWO_SM) mbar_arrive_leader(smem_addr(&tempty[set]));
          else mbar_arrive(smem_addr(&tempty[set]));
        }
      }
      float2* const out = g.partial ? g.partial + (int64_t)z * g.batch * g.M * g.N : g.out;
      const int64_t row = (int64_t)tm * C::TILE_M + rank * BM + q * 32 + lane;
      if constexpr (EPI >= 1) {
        asm volatile("bar.sync 1, 256;" ::: "memory");  // previous unit's stores done with gtab
        const int e = threadIdx.x - 64;
        const int64_t cb = (int64_t)tn * BN;
        if (e < BN) gtab[e] = (cb + e < g.N) ? map_offset(g.gmap, cb + e) : 0;
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
      if (!(g.debug & 2))
      epilogue_store<EPI, MIX>(g, out, (int64_t)b * g.M + row, row < g.M, (int64_t)tn * BN + h * 64, h * 64, mre,
                     mim, gtab, smem + C::STG_OFF + (warp - 2) * C::STG_WARP);
    }
  }
  __syncwarp();
  tc_fence_before();
  if constexpr (TWO_SM) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if constexpr (TWO_SM)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode(char* err, size_t errlen) {
  static EncodeTiledFn fn = nullptr;
  if (fn) return fn;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(e));
    return nullptr;
  }
  fn = reinterpret_cast<EncodeTiledFn>(p);
  return fn;
}

int encode_planes(void* tmap, const float* base, int64_t rows_total, int64_t kp, int box_rows,
                  char* err, size_t errlen, int nplanes = 4) {
  EncodeTiledFn enc = get_encode(err, errlen);
  if (!enc) return 1;
  // K-blocked planes [plane][kp/16][rows][16]: every box is one contiguous
  // block of box_rows x 64 B (rows past `rows` are zero-filled).
  cuuint64_t dims[3] = {(cuuint64_t)BK, (cuuint64_t)rows_total, (cuuint64_t)(nplanes * (kp / BK))};
  cuuint64_t strides[2] = {(cuuint64_t)(BK * 4), (cuuint64_t)(rows_total * BK * 4)};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                   const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled failed (CUresult %d, rows %lld kp %lld)", (int)r,
             (long long)rows_total, (long long)kp);
    return 1;
  }
  return 0;
}

}  // namespace

// 2-CTA pairs for tall GEMMs with enough pair tiles (TNX_GEMM_2SM=0 disables).
// Launch configuration cost model: pick (2-CTA pairs or single CTAs, split-K
// factor) minimising  waves * k-blocks per unit * t_kb  + split-K traffic,
// where waves = ceil(units / slots) over the 74 SM pairs / 148 SMs.  t_kb
// per slot: 2-CTA 256x128 tiles at full per-SM efficiency, 1-CTA 128x128 tiles
// at 0.88 of it (measured tensor-pipe 76 % vs 83-92 %).  Split-K adds the
// partials' HBM round trip ((2s+1) * M*N*8 B) and needs >= 8 k-blocks per unit,
// an even output size and a workspace <= 1 GB.  TNX_GEMM_2SM=0 forces 1-CTA.
namespace {
struct GemmConfig {
  int two_sm;
  int splits;
};
GemmConfig gemm_best_config(int64_t batch, int64_t M, int64_t N, int64_t kp, int fixed_splits) {
  static int mode = -1, model = -1;
  if (mode < 0) {
    const char* e = getenv("TNX_GEMM_2SM");
    mode = e ? atoi(e) : 1;
    const char* m = getenv("TNX_GEMM_MODEL");
    model = m ? atoi(m) : 1;
  }
  if (!model) {  // previous heuristics (A/B comparisons)
    const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * batch;
    int sp = 1;
    if (tiles < 148) sp = (int)std::max<int64_t>(1, std::min<int64_t>(148 / tiles, kp / BK / 8));
    if (fixed_splits > 0) sp = fixed_splits;
    const int64_t pair_tiles = ((M + 255) / 256) * ((N + BN - 1) / BN) * batch;
    return {mode && M >= 256 && pair_tiles >= 74 ? 1 : 0, sp};
  }
  const int64_t nkb = kp / BK;
  const double r_sm = 2.0e12;                // complex flop/s per SM (~296 TF/s / 148)
  const double hbm = 5.0e12;                 // B/s for the split-K partials
  const double per_wave = 1.0e-6;            // pipeline fill / epilogue tail per wave
  const bool even = (batch * M * N) % 2 == 0;
  GemmConfig best{0, 1};
  double best_t = 1e300;
  for (int t = 0; t <= 1; ++t) {
    if (t && (!mode || M < 256)) continue;
    const int64_t tiles = (t ? (M + 255) / 256 : (M + BM - 1) / BM) * ((N + BN - 1) / BN) * batch;
    const int64_t slots = t ? 74 : 148;
    const double tkb = 8.0 * (t ? 256 : BM) * BN * BK / (t ? 2.0 * r_sm : 0.88 * r_sm);
    // enough splits to fill two waves (few output tiles, long K), >= 8 k-blocks each
    const int64_t sfill = std::max<int64_t>(16, (2 * slots + tiles - 1) / tiles);
    const int smax = fixed_splits > 0 ? fixed_splits : (int)std::max<int64_t>(1, std::min(sfill, nkb / 8));
    for (int sp = fixed_splits > 0 ? fixed_splits : 1; sp <= smax; ++sp) {
      if (sp > 1 && (!even || 8.0 * sp * batch * M * N > 1.0e9)) break;
      const int64_t kbu = (nkb + sp - 1) / sp;
      const int64_t zs = (nkb + kbu - 1) / kbu;
      const int64_t units = tiles * zs;
      const int64_t waves = (units + slots - 1) / slots;
      double time = (double)waves * ((double)kbu * tkb + per_wave);
      if (zs > 1) time += (2.0 * zs + 1.0) * 8.0 * batch * M * N / hbm;
      if (time < best_t * (1.0 - 1e-9)) {
        best_t = time;
        best = {t, (int)zs};
      }
    }
  }
  return best;
}
}  // namespace

int gemm_stack_enabled() {
  static const int v = getenv("TNX_GEMM_STACKB") ? atoi(getenv("TNX_GEMM_STACKB")) : 1;
  return v;
}

// Stacked B pays when its MMA-time gain (~13 % of 8*M*N*K at ~300 TF/s,
// measured) exceeds the extra B-plane traffic (+8 B written by the producer
// and +8 B read per B element, ~16*N*K bytes at ~5 TB/s):  M > ~920 rows.
// Streaming-bound shapes (few A rows, e.g. M=256 with K=2^19) stay unstacked.
int gemm_use_stack(int64_t batch, int64_t M, int64_t N, int64_t kp, int two_sm) {
  (void)batch;
  (void)N;
  (void)kp;
  return two_sm && gemm_stack_enabled() && M >= 1024 ? 1 : 0;
}

int gemm_use_2sm(int64_t batch, int64_t M, int64_t N, int64_t kp, int splits) {
  return gemm_best_config(batch, M, N, kp, splits > 0 ? splits : 1).two_sm;
}

typedef void (*GemmKernelFn)(CUtensorMap, CUtensorMap, GemmArgs);

template <bool TWO_SM>
GemmKernelFn gemm_kernel_for(bool mix, int epi, bool stack = false) {
  if constexpr (TWO_SM) {
    if (stack && !mix) {
      if (epi == 2) return gemm_c64_3xtf32_kernel<true, false, 2, true>;
      if (epi == 1) return gemm_c64_3xtf32_kernel<true, false, 1, true>;
      return gemm_c64_3xtf32_kernel<true, false, 0, true>;
    }
  }
  if (mix) {
    if (epi == 2) return gemm_c64_3xtf32_kernel<TWO_SM, true, 2, false>;
    if (epi == 1) return gemm_c64_3xtf32_kernel<TWO_SM, true, 1, false>;
    return gemm_c64_3xtf32_kernel<TWO_SM, true, 0, false>;
  }
  if (epi == 2) return gemm_c64_3xtf32_kernel<TWO_SM, false, 2, false>;
  if (epi == 1) return gemm_c64_3xtf32_kernel<TWO_SM, false, 1, false>;
  return gemm_c64_3xtf32_kernel<TWO_SM, false, 0, false>;
}

int gemm_init_attributes(char* err, size_t errlen) {
  cudaError_t e = cudaSuccess;
  for (int mix = 0; mix < 2 && e == cudaSuccess; ++mix)
    for (int epi = 0; epi < 3 && e == cudaSuccess; ++epi) {
      e = cudaFuncSetAttribute(gemm_kernel_for<true>(mix, epi), cudaFuncAttributeMaxDynamicSharedMemorySize,
                               KCfg<true>::SMEM);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(gemm_kernel_for<false>(mix, epi), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 KCfg<false>::SMEM);
      if (e == cudaSuccess && !mix)
        e = cudaFuncSetAttribute(gemm_kernel_for<true>(false, epi, true),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, KCfg<true, true>::SMEM);
    }
  if (e != cudaSuccess) {
    snprintf(err, errlen, "cudaFuncSetAttribute(gemm): %s", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

int gemm_prepare(GemmPlan* g, const float* a_planes, const float* b_planes, float2* out,
                 int64_t batch, int64_t M, int64_t N, int64_t kp, int splits, float2* partial,
                 char* err, size_t errlen, int stack_b) {
  std::memset(g, 0, sizeof(*g));
  g->splits = splits;
  g->partial = partial;
  if (splits > 1 && (!partial || (batch * M * N) % 2 != 0)) {
    snprintf(err, errlen, "gemm: split-K needs a workspace and an even output size");
    return 1;
  }
  if (kp % BK != 0) {
    snprintf(err, errlen, "gemm: kp=%lld not a multiple of %d", (long long)kp, BK);
    return 1;
  }
  if (4 * batch * (M > N ? M : N) >= (int64_t(1) << 31)) {
    snprintf(err, errlen, "gemm: row coordinate exceeds int32");
    return 1;
  }
  g->two_sm = gemm_use_2sm(batch, M, N, kp, splits);
  if (stack_b && !g->two_sm) {
    snprintf(err, errlen, "gemm: stacked B needs the 2-CTA configuration");
    return 1;
  }
  g->stackb = stack_b ? 1 : 0;
  if (encode_planes(g->tmap_a, a_planes, batch * M, kp, BM, err, errlen)) return 1;
  if (encode_planes(g->tmap_b, b_planes, batch * N, kp, g->two_sm && !stack_b ? BN_HALF : BN, err, errlen,
                    stack_b ? 6 : 4))
    return 1;
  g->out = out;
  g->M = M;
  g->N = N;
  g->kp = kp;
  g->batch = batch;
  g->ok = 1;
  return 0;
}

__global__ void splitk_reduce_kernel(const float4* __restrict__ part, float4* __restrict__ out,
                                     int64_t n4, int64_t stride4, int splits) {
  pdl_wait();
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += step) {
    float4 a = part[i];
    for (int s = 1; s < splits; ++s) {
      float4 v = part[i + s * stride4];
      a.x += v.x;
      a.y += v.y;
      a.z += v.z;
      a.w += v.w;
    }
    out[i] = a;
  }
}

int gemm_choose_splits(int64_t batch, int64_t M, int64_t N, int64_t kp) {
  return gemm_best_config(batch, M, N, kp, 0).splits;
}

// k-blocks (of 16) accumulated in TMEM per promotion round; TNX_GEMM_PROMOTE
// overrides (measured trade-off: accuracy vs TMEM-pipe load of the promotion).
static int gemm_group_m() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("TNX_GEMM_GROUP_M");
    v = e ? atoi(e) : GROUP_M;
    if (v < 1) v = 1;
  }
  return v;
}

static int gemm_default_promote() {
  static int v = 0;
  if (!v) {
    const char* e = getenv("TNX_GEMM_PROMOTE");
    v = e ? atoi(e) : 3;
    if (v < 1) v = 1;
  }
  return v;
}

cudaError_t launch_gemm(const GemmPlan& g, cudaStream_t st) {
  GemmArgs a;
  a.out = g.out;
  a.M = g.M;
  a.N = g.N;
  a.batch = g.batch;
  a.num_kb = (int32_t)(g.kp / BK);
  a.tiles_m = (int32_t)((g.M + BM - 1) / BM);
  a.tiles_n = (int32_t)((g.N + BN - 1) / BN);
  a.promote = g.promote > 0 ? g.promote : gemm_default_promote();
  a.direct = g.direct;
  a.dvec = g.dvec;
  a.mix = g.mix;
  a.dmix = g.dmix;
  a.dside = g.dside;
  a.dplanes = g.dplanes;
  a.dplane_stride = g.dplane_stride;
  a.fmap = g.fmap;
  a.gmap = g.gmap;
  a.group_m = gemm_group_m();
  {
    static const int dbg = getenv("TNX_GEMM_DEBUG") ? atoi(getenv("TNX_GEMM_DEBUG")) : 0;
    a.debug = dbg;
    a.dstack = g.dstack;
    a.dpair = g.dpair;
    static const int snake = getenv("TNX_GEMM_KSNAKE") ? atoi(getenv("TNX_GEMM_KSNAKE")) : 1;
    a.ksnake = snake;
    // a unit's first TMEM round spans TNX_GEMM_FIRST (default 6) k-blocks, later
    // rounds `promote`: while the epilogue warps store the previous unit, the
    // MMA can run two rounds ahead, and a long first round lets that cover a
    // mid-K unit's stores (cfg4 GEMM time -1.1 %; only the first round's
    // accumulation gets longer, so long-K accuracy is unchanged)
    static const int first = getenv("TNX_GEMM_FIRST") ? atoi(getenv("TNX_GEMM_FIRST")) : 6;
    a.first = g.promote > 0 ? 0 : first;
    // kappa of the round-toward-zero compensation (TNX_GEMM_RZC; 0 disables).
    // Measured (tools/gemm_bias.py, tools/prefix_parity.py): the
    // bias that nulls it is ~0.6 on random CN(0,1) operands and ~0.35 on the
    // circuit workloads (structured operands often sum exactly, so fewer
    // truncations lose bits).  0.35 removes the circuits' bias and 60 % of the
    // random-data bias; on data whose sums are all exact it over-corrects by
    // at most 0.35 * 2^-24 * (6 n_kb - 2) per GEMM (< 7.1e-7 for a 6-k-block
    // round), below the uncompensated bias on random data.
    static const float kappa = getenv("TNX_GEMM_RZC") ? (float)atof(getenv("TNX_GEMM_RZC")) : 0.35f;
    a.rz_kappa = kappa;
    static const int l2hint = getenv("TNX_GEMM_L2HINT") ? atoi(getenv("TNX_GEMM_L2HINT")) : 1;
    a.l2keep = l2hint & 1;
    a.stcs = (l2hint >> 1) & 1;
  }
  const int splits = g.splits > 1 ? g.splits : 1;
  a.kb_per_split = (a.num_kb + splits - 1) / splits;
  a.partial = splits > 1 ? g.partial : nullptr;
  a.rows_a = g.batch * g.M;
  a.rows_b = g.batch * g.N;
  const int zs = (a.num_kb + a.kb_per_split - 1) / a.kb_per_split;
  a.splits = zs;
  // Optional (TNX_GEMM_ADAPT=n): short units (few k-blocks) fit in two TMEM
  // rounds (interval up to n) so their stores overlap the next unit's MMAs
  // fully -- the epilogue warps store a unit while the MMA can run at most two
  // rounds ahead.  Measured on cfg4: -0.35 % GEMM time for +20 % error on the
  // depth-20 amplitude, so off by default.  TNX_GEMM_PROMOTE pins the interval.
  if (g.promote <= 0 && !getenv("TNX_GEMM_PROMOTE")) {
    static const int adapt = getenv("TNX_GEMM_ADAPT") ? atoi(getenv("TNX_GEMM_ADAPT")) : 0;
    const int kbu = a.kb_per_split;
    if (kbu > 2 * a.promote && kbu <= 2 * adapt) a.promote = (kbu + 1) / 2;
  }
  const CUtensorMap* ta = reinterpret_cast<const CUtensorMap*>(g.tmap_a);
  const CUtensorMap* tb = reinterpret_cast<const CUtensorMap*>(g.tmap_b);
  const int epi = a.direct ? (a.dvec ? 2 : 1) : 0;
  if (g.direct && g.dmix != g.mix) return cudaErrorInvalidValue;  // planes follow the plan's precision
  if (g.stackb && (g.mix || !g.two_sm)) return cudaErrorInvalidValue;
  if (g.two_sm) a.tiles_m = (int32_t)((g.M + 255) / 256);
  const int64_t units = (int64_t)a.tiles_m * a.tiles_n * g.batch * zs;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int nattr = 0;
  if (pdl_enabled()) {
    attr[nattr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[nattr].val.programmaticStreamSerializationAllowed = 1;
    ++nattr;
  }
  cfg.attrs = attr;
  if (g.two_sm) {
    // TNX_GEMM_MAXPAIRS caps the persistent grid (diagnostics: per-SM vs chip-wide limits)
    static const int64_t maxpairs = getenv("TNX_GEMM_MAXPAIRS") ? atoll(getenv("TNX_GEMM_MAXPAIRS")) : 74;
    const int64_t clusters = std::min<int64_t>(units, std::max<int64_t>(1, std::min<int64_t>(74, maxpairs)));
    cfg.gridDim = dim3((unsigned)(2 * clusters));
    cfg.dynamicSmemBytes = g.stackb ? KCfg<true, true>::SMEM : KCfg<true>::SMEM;
    attr[nattr].id = cudaLaunchAttributeClusterDimension;
    attr[nattr].val.clusterDim.x = 2;
    attr[nattr].val.clusterDim.y = 1;
    attr[nattr].val.clusterDim.z = 1;
    cfg.numAttrs = nattr + 1;
    cudaError_t le = cudaLaunchKernelEx(&cfg, gemm_kernel_for<true>(a.mix != 0, epi, g.stackb != 0), *ta, *tb, a);
    if (le != cudaSuccess) return le;
  } else {
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(units, 148));
    cfg.dynamicSmemBytes = KCfg<false>::SMEM;
    cfg.numAttrs = nattr;
    cudaError_t le = cudaLaunchKernelEx(&cfg, gemm_kernel_for<false>(a.mix != 0, epi), *ta, *tb, a);
    if (le != cudaSuccess) return le;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || zs == 1) return e;
  const int64_t n = g.batch * g.M * g.N;  // complex elements
  if (n % 2 != 0) return cudaErrorInvalidValue;
  const int64_t n4 = n / 2;
  int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 148 * 16);
  launch_pdl(splitk_reduce_kernel, blocks, 256, 0, st, reinterpret_cast<const float4*>(g.partial),
                                               reinterpret_cast<float4*>(g.out), n4, n4, zs);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Tensor-pipe ceiling: an MMA-only loop (no TMA, no promotion, no epilogue)
// over operands resident in shared memory, one CTA (or CTA pair) per SM.
// Issues `iters` tcgen05.mma of N=256 (M=128 per CTA, M=256 per pair with
// cta_group::2) alternating between two TMEM accumulator sets and two k-steps
// of the same SWIZZLE_64B tiles the GEMM uses, so the per-MMA shared-memory
// operand reads match the stacked-B GEMM's.  Operands are pseudo-random
// (realistic switching power).  Each CTA records its clock64 and globaltimer
// deltas, giving the SM clock the ceiling was measured at.
namespace {
constexpr int PEAK_THREADS = 128;
constexpr int PEAK_A = BM * BK * 4;     // 8 KB: 128 rows x 64 B
constexpr int PEAK_B = 2 * BN * BK * 4; // 16 KB: up to 256 rows x 64 B
constexpr int PEAK_SMEM = 200 * 1024;   // one CTA per SM

__device__ __forceinline__ uint32_t peak_hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

template <bool TWO_SM, bool BF16>
__global__ void __launch_bounds__(PEAK_THREADS, 1)
    mma_peak_kernel(int64_t iters, unsigned long long* rec) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* done = reinterpret_cast<uint64_t*>(smem + PEAK_A + PEAK_B);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const uint32_t rank = TWO_SM ? cluster_rank() : 0u;
  // pseudo-random operands in [-1, 1): fp32 bits, or bf16 pairs
  for (int i = threadIdx.x; i < (PEAK_A + PEAK_B) / 4; i += PEAK_THREADS) {
    const uint32_t h = peak_hash((uint32_t)i * 2654435761u + blockIdx.x * 97u + 1u);
    uint32_t v;
    if (BF16) {
      const float lo = (float)(int)(h & 0xffffu) / 32768.0f - 1.0f;
      const float hi = (float)(int)(h >> 16) / 32768.0f - 1.0f;
      v = (__float_as_uint(lo) >> 16) | (__float_as_uint(hi) & 0xffff0000u);
    } else {
      v = __float_as_uint((float)(int)(h >> 8) / 8388608.0f - 1.0f);
    }
    reinterpret_cast<uint32_t*>(smem)[i] = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    if constexpr (TWO_SM) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_addr(tmem_slot)), "r"(TMEM_COLS) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_addr(tmem_slot)), "r"(TMEM_COLS) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (threadIdx.x == 32) {
    mbar_init(smem_addr(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  if constexpr (TWO_SM) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  unsigned long long c0 = clock64(), g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  if (threadIdx.x == 32 && rank == 0) {
    constexpr uint32_t ID = idesc_mma<TWO_SM>(false, BF16 ? 1u : 2u, 2 * BN);
    const uint32_t sa = smem_addr(smem), sb = smem_addr(smem + PEAK_A);
    for (int64_t i = 0; i < iters; ++i) {
      const uint32_t koff = (uint32_t)(i & 1) * 32u;
      const uint32_t d = tmem_base + (uint32_t)((i >> 1) & 1) * 256u;
      const uint32_t acc = i >= 4 ? 1u : 0u;
      const uint64_t a = umma_desc_sw64(sa + koff), b = umma_desc_sw64(sb + koff);
      if constexpr (TWO_SM) {
        if (BF16) umma_bf16_2sm(d, a, b, ID, acc); else umma_tf32_2sm(d, a, b, ID, acc);
      } else {
        if (BF16) umma_bf16(d, a, b, ID, acc); else umma_tf32(d, a, b, ID, acc);
      }
    }
    if constexpr (TWO_SM) umma_commit_2sm(smem_addr(done)); else umma_commit(smem_addr(done));
  }
  if (threadIdx.x == 0) mbar_wait(smem_addr(done), 0);
  __syncthreads();
  tc_fence_after();
  const unsigned long long c1 = clock64();
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0) {
    rec[2 * blockIdx.x] = c1 - c0;
    rec[2 * blockIdx.x + 1] = g1 - g0;
  }
  tc_fence_before();
  if constexpr (TWO_SM) cluster_sync_all(); else __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if constexpr (TWO_SM)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
  }
}

// FP32 SIMT ceiling: 8 independent FFMA chains per thread, 4 x 256 threads per
// SM; the result is folded into rec so the chains are live.
__global__ void __launch_bounds__(256) ffma_peak_kernel(int64_t iters, unsigned long long* rec) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = 1.0f + 1e-7f * (float)(threadIdx.x + j);
  const float b = 0.999999f, c = 1e-7f;
  unsigned long long c0 = clock64(), g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += a[j];
  const unsigned long long c1 = clock64();
  unsigned long long g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && (blockIdx.x & 3) == 0) {
    rec[2 * (blockIdx.x >> 2)] = (c1 - c0) + (acc == 12345.f ? 1ull : 0ull);
    rec[2 * (blockIdx.x >> 2) + 1] = g1 - g0;
  }
}

template <bool TWO_SM, bool BF16>
cudaError_t launch_mma_peak(int64_t iters, unsigned long long* rec, int grid, cudaStream_t st) {
  auto k = mma_peak_kernel<TWO_SM, BF16>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PEAK_SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(PEAK_THREADS);
  cfg.dynamicSmemBytes = PEAK_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = TWO_SM ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = TWO_SM ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, k, iters, rec);
  return e != cudaSuccess ? e : cudaGetLastError();
}
}  // namespace

int gemm_mma_peak(int kind, int two_sm, int64_t iters, cudaStream_t st, double* tflops, double* sm_mhz,
                  double* ms, char* err, size_t errlen) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool ffma = kind == 2;
  const int bf16 = kind == 1;
  const int grid = ffma ? sms : two_sm ? (sms / 2) * 2 : sms;
  unsigned long long* rec = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaError_t e = cudaMalloc(&rec, sizeof(unsigned long long) * 2 * grid);
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  auto launch = [&](int64_t n) {
    if (ffma) {
      ffma_peak_kernel<<<4 * sms, 256, 0, st>>>(n, rec);
      return cudaGetLastError();
    }
    if (two_sm) return bf16 ? launch_mma_peak<true, true>(n, rec, grid, st) : launch_mma_peak<true, false>(n, rec, grid, st);
    return bf16 ? launch_mma_peak<false, true>(n, rec, grid, st) : launch_mma_peak<false, false>(n, rec, grid, st);
  };
  float t = 0.f;
  if (e == cudaSuccess) e = launch(std::min<int64_t>(iters, 4096));  // warm-up
  if (e == cudaSuccess) e = cudaEventRecord(e0, st);
  if (e == cudaSuccess) e = launch(iters);
  if (e == cudaSuccess) e = cudaEventRecord(e1, st);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  if (e == cudaSuccess) e = cudaEventElapsedTime(&t, e0, e1);
  std::vector<unsigned long long> h(2 * grid);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), rec, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  if (rec) cudaFree(rec);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (e != cudaSuccess) {
    snprintf(err, errlen, "mma peak: %s", cudaGetErrorString(e));
    return 1;
  }
  // flop per MMA per CTA: 2 * 128 rows * 256 columns * K (8 tf32 / 16 bf16);
  // FFMA: 2 flop x 8 chains per thread per iteration, 4 x 256 threads per SM
  const double flop = ffma ? (double)sms * 1024.0 * (double)iters * 16.0
                           : (double)grid * (double)iters * 2.0 * BM * 2 * BN * (bf16 ? 16 : 8);
  *ms = t;
  *tflops = flop / (t * 1e-3) / 1e12;
  std::vector<double> mhz;
  for (int i = 0; i < grid; ++i)
    if (h[2 * i + 1] > 0) mhz.push_back(1e3 * (double)h[2 * i] / (double)h[2 * i + 1]);
  std::sort(mhz.begin(), mhz.end());
  *sm_mhz = mhz.empty() ? 0.0 : mhz[mhz.size() / 2];
  return 0;
}

}  // namespace tnx
