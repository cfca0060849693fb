// Memory-bound kernels of the sliced contraction executor (sm_100a).  Every
// kernel starts with griddepcontrol.wait (programmatic dependent launch).
//
//  K1 gather  : fix_index of every slice-dependent leaf for the current slice
//               id (reference dense.py:161-170), read from a device counter so
//               the per-slice CUDA graph needs no host update; one launch, block
//               ranges per leaf, contiguous runs merged, 16 B copies.
//  K4 simt    : strided pairwise contraction (reference pairwise_contract,
//               dense.py:61-76) in FP32 complex: all thread/warp-mode vertices
//               of a dependency level in one batched launch (2^lg lanes per
//               output), split mode (block partials + FP64 finalize) for long
//               sums; strided fast path with 16 B loads.
//  K2 pack / permute : complex64 -> split-TF32 planes the tcgen05 GEMM consumes,
//               K-blocked [kp/16][rows][16]; shared-memory tiled, pipelined
//               permute (`perm_vec_kernel`), gather fallback (`pack_kernel`);
//               mode 5 fuses a full contraction (permute + dot).
//  K5 dot     : streaming complex dot for equal layouts.
//  K6 accum   : root -> tn.output order, Kahan-compensated complex128
//               accumulation across slices; allreduce_kernel sums
//               several plans' accumulators (tnx_allreduce).
#include <climits>
#include <cstdlib>
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include "tnx_kernels.h"

namespace tnx {

__device__ __forceinline__ void decode2(const IdxMap& m, int64_t idx, int64_t& o0, int64_t& o1) {
#pragma unroll 1
  for (int i = m.n - 1; i >= 0; --i) {
    int64_t r;
    if (m.lg[i] >= 0) {
      r = idx & (m.dim[i] - 1);
      idx >>= m.lg[i];
    } else {
      int64_t q = idx / m.dim[i];
      r = idx - q * m.dim[i];
      idx = q;
    }
    o0 += r * m.st0[i];
    o1 += r * m.st1[i];
  }
}

__device__ __forceinline__ void decode1(const IdxMap& m, int64_t idx, int64_t& o0) {
#pragma unroll 1
  for (int i = m.n - 1; i >= 0; --i) {
    int64_t r;
    if (m.lg[i] >= 0) {
      r = idx & (m.dim[i] - 1);
      idx >>= m.lg[i];
    } else {
      int64_t q = idx / m.dim[i];
      r = idx - q * m.dim[i];
      idx = q;
    }
    o0 += r * m.st0[i];
  }
}

__device__ __forceinline__ void cfma(float2& acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}

// ------------------------------------------------------------------ gather
// One launch for all slice-dependent leaves: each job owns a contiguous range of
// blocks (prefix table `start`, sized on the host in proportion to the leaf
// slice), so one large leaf is spread over the whole GPU while tiny circuit
// leaves take one block each.  Kept dims are pre-merged into contiguous runs.
__global__ void __launch_bounds__(256) gather_kernel(const GatherJob* __restrict__ jobs,
                                                     const int32_t* __restrict__ start, int njobs,
                                                     const float2* __restrict__ pool,
                                                     const unsigned long long* __restrict__ counter) {
  pdl_wait();
  int lo = 0, hi = njobs - 1;
  const int b = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  const GatherJob& j = jobs[lo];
  const int lb = b - start[lo];
  const int nb = start[lo + 1] - start[lo];
  const unsigned long long s = *counter;
  int64_t base = j.src;
  for (int i = 0; i < j.n_sl; ++i) {
    unsigned long long digit = (s / j.radix[i]) % (unsigned long long)j.sdim[i];
    base += (int64_t)digit * j.sst[i];
  }
  const int nk = j.n_kept;
  const int64_t inner = nk > 0 ? j.kdim[nk - 1] : 1;
  const int64_t inner_st = nk > 0 ? j.kst[nk - 1] : 0;
  if (j.vec) {  // element pairs: the inner run has unit stride and even length
    const int64_t half = inner >> 1;
    float4* dst4 = reinterpret_cast<float4*>(j.dst);
    for (int64_t e = (int64_t)lb * blockDim.x + threadIdx.x; e < (j.out_size >> 1);
         e += (int64_t)nb * blockDim.x) {
      int64_t idx = e / half;
      int64_t off = base + 2 * (e - idx * half);
      for (int i = nk - 2; i >= 0; --i) {
        const int64_t q = idx / j.kdim[i];
        off += (idx - q * j.kdim[i]) * j.kst[i];
        idx = q;
      }
      __stcs(dst4 + e, __ldcs(reinterpret_cast<const float4*>(pool + off)));
    }
    return;
  }
  for (int64_t e = (int64_t)lb * blockDim.x + threadIdx.x; e < j.out_size; e += (int64_t)nb * blockDim.x) {
    int64_t idx = e / inner;
    int64_t off = base + (e - idx * inner) * inner_st;
    for (int i = nk - 2; i >= 0; --i) {
      const int64_t q = idx / j.kdim[i];
      off += (idx - q * j.kdim[i]) * j.kst[i];
      idx = q;
    }
    j.dst[e] = pool[off];
  }
}

cudaError_t launch_gather(const GatherJob* jobs, const int32_t* start, int njobs, int total_blocks,
                          const float2* pool, const unsigned long long* counter, cudaStream_t st) {
  if (njobs == 0) return cudaSuccess;
  launch_pdl(gather_kernel, total_blocks, 256, 0, st, jobs, start, njobs, pool, counter);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ simt
// Summed-index loop shared by the SIMT kernels: lanes lane0, lane0 + step, ...
// of [j0, j1).  Fast path when the summed labels merge into one strided run
// (no decode / table; unrolled so independent loads overlap).
__device__ __forceinline__ void simt_sum(const SimtParams& p, int64_t ox, int64_t oy, int64_t j0, int64_t j1,
                                         int64_t step, float2& acc) {
  if (p.sum.n <= 1) {
    const int64_t s0 = p.sum.n ? p.sum.st0[0] : 0, s1 = p.sum.n ? p.sum.st1[0] : 0;
    const float2* __restrict__ xp = p.x + ox;
    const float2* __restrict__ yp = p.y + oy;
    float2 a2 = make_float2(0.f, 0.f);
    int64_t j = j0;
    if (step == 1 && s0 == 1 && s1 == 1 && ((ox | oy | j0) & 1) == 0) {
      // contiguous run in both operands: 16-byte loads (two complex values)
      for (; j + 1 < j1; j += 2) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(xp + j));
        const float4 yv = __ldg(reinterpret_cast<const float4*>(yp + j));
        cfma(acc, make_float2(xv.x, xv.y), make_float2(yv.x, yv.y));
        cfma(a2, make_float2(xv.z, xv.w), make_float2(yv.z, yv.w));
      }
    }
    for (; j + step < j1; j += 2 * step) {
      const float2 x0 = __ldg(xp + j * s0), y0 = __ldg(yp + j * s1);
      const float2 x1 = __ldg(xp + (j + step) * s0), y1 = __ldg(yp + (j + step) * s1);
      cfma(acc, x0, y0);
      cfma(a2, x1, y1);
    }
    if (j < j1) cfma(acc, __ldg(xp + j * s0), __ldg(yp + j * s1));
    acc.x += a2.x;
    acc.y += a2.y;
  } else if (p.sum_tab) {
    for (int64_t j = j0; j < j1; j += step) {
      const Int2Off t = p.sum_tab[j];
      cfma(acc, p.x[ox + t.x], p.y[oy + t.y]);
    }
  } else {
    for (int64_t j = j0; j < j1; j += step) {
      int64_t sx = ox, sy = oy;
      decode2(p.sum, j, sx, sy);
      cfma(acc, p.x[sx], p.y[sy]);
    }
  }
}

__global__ void __launch_bounds__(256) simt_split_kernel(const SimtParams p) {
  pdl_wait();
  // grid: (nsplit, out_size)
  const int64_t o = blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * p.chunk;
  const int64_t j1 = min(j0 + p.chunk, p.sum_size);
  int64_t ox = 0, oy = 0;
  decode2(p.out, o, ox, oy);
  float2 acc = make_float2(0.f, 0.f);
  simt_sum(p, ox, oy, j0 + threadIdx.x, j1, blockDim.x, acc);
  __shared__ float2 red[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    int nw = blockDim.x >> 5;
    float2 v = threadIdx.x < nw ? red[threadIdx.x] : make_float2(0.f, 0.f);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
      v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
    }
    if (threadIdx.x == 0) p.partial[o * p.nsplit + blockIdx.x] = v;
  }
}

__global__ void simt_finalize_kernel(const float2* __restrict__ partial, float2* __restrict__ z,
                                     int64_t out_size, int nsplit) {
  pdl_wait();
  const int64_t o = blockIdx.x;
  double re = 0.0, im = 0.0;
  for (int i = threadIdx.x; i < nsplit; i += blockDim.x) {
    float2 v = partial[o * nsplit + i];
    re += v.x;
    im += v.y;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, off);
    im += __shfl_xor_sync(0xffffffffu, im, off);
  }
  __shared__ double r2[64];
  if ((threadIdx.x & 31) == 0) {
    r2[threadIdx.x >> 5] = re;
    r2[32 + (threadIdx.x >> 5)] = im;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      a += r2[w];
      b += r2[32 + w];
    }
    z[o] = make_float2((float)a, (float)b);
  }
}

static int grid_for(int64_t work, int threads, int max_blocks) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

cudaError_t launch_simt(const SimtParams& p, cudaStream_t st) {
  if (p.out_size == 0) return cudaSuccess;
  // thread / warp modes run batched per dependency level (launch_simt_batch)
  if (p.mode != SIMT_SPLIT) return cudaErrorInvalidValue;
  {
    dim3 grid((unsigned)p.nsplit, (unsigned)p.out_size);
    launch_pdl(simt_split_kernel, grid, 256, 0, st, p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    launch_pdl(simt_finalize_kernel, (unsigned)p.out_size, 128, 0, st, p.partial, p.z, p.out_size, p.nsplit);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ batched simt
__global__ void __launch_bounds__(256) simt_batch_kernel(const SimtParams* __restrict__ jobs,
                                                         const int32_t* __restrict__ start, int njobs) {
  pdl_wait();
  // locate this block's job (binary search over the block prefix)
  int lo = 0, hi = njobs - 1;
  const int b = blockIdx.x;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= b) lo = mid;
    else hi = mid - 1;
  }
  const SimtParams& p = jobs[lo];
  const int lb = b - start[lo];
  const int nb = start[lo + 1] - start[lo];
  // 2^lg lanes cooperate on one output (0: thread mode, 5: warp mode); the loop
  // is warp-uniform so the group reductions are legal shuffles
  const int lg = p.group_lg;
  const int G = 1 << lg;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int per_warp = 32 >> lg;
  const int64_t w0 = ((int64_t)lb * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)nb * blockDim.x) >> 5;
  for (int64_t base = w0 * per_warp; base < p.out_size; base += nw * per_warp) {
    const int64_t o = base + (lane >> lg);
    const bool valid = o < p.out_size;
    float2 acc = make_float2(0.f, 0.f);
    if (valid) {
      int64_t ox = 0, oy = 0;
      decode2(p.out, o, ox, oy);
      simt_sum(p, ox, oy, gl, p.sum_size, G, acc);
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (valid && gl == 0) {
      if (p.znp > 0) {
        // SIMT -> GEMM fusion: the parent GEMM's split-TF32 operand planes
        int64_t off = 0;
        decode1(p.zmap, o, off);
        float* d = p.zplanes + off;
        const float rh = tf32_hi(acc.x), ih = tf32_hi(acc.y);
        const float rl = tf32_lo(acc.x, rh), il = tf32_lo(acc.y, ih);
        d[0] = rh;
        d[p.zps] = rl;
        d[2 * p.zps] = ih;
        d[3 * p.zps] = il;
        if (p.znp == 6) {
          d[4 * p.zps] = -ih;
          d[5 * p.zps] = -il;
        }
      } else {
        p.z[o] = acc;
      }
    }
  }
}

int simt_blocks(const SimtParams& p) {
  const int64_t work = p.out_size << p.group_lg;
  int64_t b = (work + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

cudaError_t launch_simt_batch(const SimtParams* jobs, const int32_t* block_start, int njobs,
                              int total_blocks, cudaStream_t st) {
  if (njobs == 0) return cudaSuccess;
  launch_pdl(simt_batch_kernel, total_blocks, 256, 0, st, jobs, block_start, njobs);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ pack
__global__ void __launch_bounds__(256) pack_kernel(const PackParams p) {
  pdl_wait();
  // destination planes are K-blocked: offset(r, k) = ((k / 16) * rows + r) * 16 + k % 16
  const int64_t total = p.rows * p.kp;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t ki = e & 15;
    const int64_t q = e >> 4;
    const int64_t kb = q / p.rows;
    const int64_t r = q - kb * p.rows;
    const int64_t k = kb * 16 + ki;
    float re = 0.f, im = 0.f;
    if (k < p.K) {
      int64_t off = 0;
      decode1(p.row, r, off);
      decode1(p.col, k, off);
      float2 v = p.src[off];
      re = v.x;
      im = v.y;
    }
    const float re_hi = tf32_hi(re);
    const float im_hi = tf32_hi(im);
    p.dst[e] = re_hi;
    p.dst[e + 2 * p.plane_stride] = im_hi;
    if (p.mix) {
      store_mix_x(p.dst + p.plane_stride, e, re, p.mix == 2);
      store_mix_x(p.dst + 3 * p.plane_stride, e, im, p.mix == 2);
    } else {
      const float im_lo = tf32_lo(im, im_hi);
      p.dst[e + p.plane_stride] = tf32_lo(re, re_hi);
      p.dst[e + 3 * p.plane_stride] = im_lo;
      if (p.nplanes == 6) {  // stacked-B operand: negated imaginary planes
        p.dst[e + 4 * p.plane_stride] = -im_hi;
        p.dst[e + 5 * p.plane_stride] = -im_lo;
      }
    }
  }
}

cudaError_t launch_pack(const PackParams& p, cudaStream_t st) {
  launch_pdl(pack_kernel, grid_for(p.rows * p.kp, 256, 148 * 32), 256, 0, st, p);
  return cudaGetLastError();
}

// block reduction of the fused perm-dot partial sums -> partial[blockIdx.x]
__device__ __forceinline__ void perm_dot_reduce(float re, float im, float2* partial) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, off);
    im += __shfl_xor_sync(0xffffffffu, im, off);
  }
  __shared__ float2 red[8];
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_float2(re, im);
  __syncthreads();
  if (threadIdx.x == 0) {
    float2 v = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      v.x += red[w].x;
      v.y += red[w].y;
    }
    partial[blockIdx.x] = v;
  }
}

// ------------------------------------------------------------------ tiled permute
__global__ void __launch_bounds__(256) perm_kernel(const PermParams p) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char perm_smem[];
  __shared__ int64_t base_s[64], base_d[64];
  const int ts = p.ts;
  const int G = p.group;
  int32_t* t_src = reinterpret_cast<int32_t*>(perm_smem);
  int32_t* t_idx = t_src + ts;
  int32_t* t_dst = t_idx + ts;
  float2* tile = reinterpret_cast<float2*>(perm_smem + ((size_t)(3 * ts * 4 + 15) & ~(size_t)15));
  for (int i = threadIdx.x; i < 3 * ts; i += blockDim.x) t_src[i] = p.tab[i];
  const int64_t nchunks = (p.n_outer + G - 1) / G;
  float dre = 0.f, dim = 0.f;  // mode 5 partial sums
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int64_t o0 = c * G;
    const int gcount = (int)(p.n_outer - o0 < (int64_t)G ? p.n_outer - o0 : (int64_t)G);
    if (threadIdx.x < gcount) {
      int64_t sb = 0, db = 0;
      decode2(p.outer, o0 + threadIdx.x, sb, db);
      base_s[threadIdx.x] = sb;
      base_d[threadIdx.x] = db;
    }
    __syncthreads();
    // load: source iteration order (innermost source labels fastest)
    for (int e = threadIdx.x; e < gcount * ts; e += blockDim.x) {
      const int j = e / ts, t = e - j * ts;
      tile[j * ts + t_idx[t]] = p.src[base_s[j] + t_src[t]];
    }
    __syncthreads();
    // store: destination order (innermost destination labels fastest)
    for (int e = threadIdx.x; e < gcount * ts; e += blockDim.x) {
      const int j = e / ts, t = e - j * ts;
      const float2 v = tile[j * ts + t];
      const int64_t off = base_d[j] + t_dst[t];
      if (p.mode == 5) {
        const float2 xv = __ldg(p.dotx + off);
        dre = fmaf(xv.x, v.x, dre);
        dre = fmaf(-xv.y, v.y, dre);
        dim = fmaf(xv.x, v.y, dim);
        dim = fmaf(xv.y, v.x, dim);
        continue;
      }
      if (p.mode == 0) {
        static_cast<float2*>(p.dst)[off] = v;
      } else {
        float* d = static_cast<float*>(p.dst);
        const float re_hi = tf32_hi(v.x);
        const float im_hi = tf32_hi(v.y);
        const float im_lo = tf32_lo(v.y, im_hi);
        d[off] = re_hi;
        d[off + p.plane_stride] = tf32_lo(v.x, re_hi);
        d[off + 2 * p.plane_stride] = im_hi;
        d[off + 3 * p.plane_stride] = im_lo;
        if (p.mode == 2) {
          d[off + 4 * p.plane_stride] = -im_hi;
          d[off + 5 * p.plane_stride] = -im_lo;
        }
      }
    }
    __syncthreads();
  }
  if (p.mode == 5) perm_dot_reduce(dre, dim, p.partial);
}

// Vectorised variant: element pairs (t, t+1) are contiguous and 16 B / 8 B
// aligned in source and destination, ts is a power of two.  Software-pipelined:
// the global loads of chunk c+1 are issued into registers before chunk c is
// stored, so every SM keeps loads in flight through the store phase.  The tile
// is XOR-swizzled on float2 bits 1..3 (pairs stay adjacent and 16 B aligned, so
// the store side reads float4) to spread the transposed writes over the banks.
__device__ __forceinline__ int perm_swz(int i) {
  return i ^ ((((i >> 4) ^ (i >> 7) ^ (i >> 10)) & 7) << 1);
}

constexpr int kPermMaxPairs = 4;  // (ts * group / 2) / 256 <= 2048 / 2 / 256 (vec needs ts <= 2048)

template <bool DOT>
__global__ void __launch_bounds__(256, DOT ? 3 : 4) perm_vec_kernel(const PermParams p) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char perm_smem[];
  __shared__ int64_t base_s[2][64], base_d[2][64];
  const int ts = p.ts;
  const int lg = p.ts_log2;
  const int G = p.group;
  int32_t* t_src = reinterpret_cast<int32_t*>(perm_smem);
  int32_t* t_idx = t_src + ts;
  int32_t* t_dst = t_idx + ts;
  float2* tile = reinterpret_cast<float2*>(perm_smem + ((size_t)(3 * ts * 4 + 15) & ~(size_t)15));
  for (int i = threadIdx.x; i < 3 * ts; i += blockDim.x) t_src[i] = p.tab[i];
  const int64_t nchunks = (p.n_outer + G - 1) / G;
  const int half_mask = (ts >> 1) - 1;
  const int half_lg = lg - 1;
  float* d = static_cast<float*>(p.dst);
  auto count_of = [&](int64_t c) {
    const int64_t o0 = c * G;
    return (int)(p.n_outer - o0 < (int64_t)G ? p.n_outer - o0 : (int64_t)G);
  };
  auto bases = [&](int64_t c, int buf) {
    if (threadIdx.x < count_of(c)) {
      int64_t sb = 0, db = 0;
      decode2(p.outer, c * G + threadIdx.x, sb, db);
      base_s[buf][threadIdx.x] = sb;
      base_d[buf][threadIdx.x] = db;
    }
  };
  float4 r[kPermMaxPairs];
  auto issue = [&](int buf, int npairs) {
#pragma unroll
    for (int i = 0; i < kPermMaxPairs; ++i) {
      const int e = threadIdx.x + i * 256;
      if (e < npairs) {
        const int j = e >> half_lg, t = (e & half_mask) << 1;
        r[i] = __ldg(reinterpret_cast<const float4*>(p.src + base_s[buf][j] + t_src[t]));
      }
    }
  };
  int64_t c = blockIdx.x;
  if (c >= nchunks) return;
  float dre = 0.f, dim = 0.f;  // mode 5 partial sums
  int buf = 0;
  bases(c, 0);
  __syncthreads();
  int npairs = count_of(c) << half_lg;
  issue(0, npairs);
  while (true) {
#pragma unroll
    for (int i = 0; i < kPermMaxPairs; ++i) {
      const int e = threadIdx.x + i * 256;
      if (e < npairs) {
        const int j = e >> half_lg, t = (e & half_mask) << 1;
        tile[perm_swz((j << lg) + t_idx[t])] = make_float2(r[i].x, r[i].y);
        tile[perm_swz((j << lg) + t_idx[t + 1])] = make_float2(r[i].z, r[i].w);
      }
    }
    // fused dot: this chunk's x values (destination order, same e -> (j, t) map as
    // the store phase) go in flight now, across the barrier and the next issue
    float4 xr[kPermMaxPairs];
    if constexpr (DOT) {
#pragma unroll
      for (int i = 0; i < kPermMaxPairs; ++i) {
        const int e = threadIdx.x + i * 256;
        if (e < npairs) {
          const int j = e >> half_lg, t = (e & half_mask) << 1;
          xr[i] = __ldcs(reinterpret_cast<const float4*>(p.dotx + base_d[buf][j] + t_dst[t]));
        }
      }
    }
    const int64_t cn = c + gridDim.x;
    const bool more = cn < nchunks;
    if (more) bases(cn, buf ^ 1);
    __syncthreads();
    const int np_cur = npairs;
    if (more) {
      npairs = count_of(cn) << half_lg;
      issue(buf ^ 1, npairs);
    }
    if constexpr (DOT) {  // fused dot: multiply the permuted tile with x in place
#pragma unroll
      for (int i = 0; i < kPermMaxPairs; ++i) {
        const int e = threadIdx.x + i * 256;
        if (e < np_cur) {
          const int j = e >> half_lg, t = (e & half_mask) << 1;
          const float4 v = *reinterpret_cast<const float4*>(tile + perm_swz((j << lg) + t));
          const float4 xv = xr[i];
          dre = fmaf(xv.x, v.x, dre);
          dre = fmaf(-xv.y, v.y, dre);
          dim = fmaf(xv.x, v.y, dim);
          dim = fmaf(xv.y, v.x, dim);
          dre = fmaf(xv.z, v.z, dre);
          dre = fmaf(-xv.w, v.w, dre);
          dim = fmaf(xv.z, v.w, dim);
          dim = fmaf(xv.w, v.z, dim);
        }
      }
    }
    for (int e = threadIdx.x; !DOT && e < np_cur; e += blockDim.x) {
      const int j = e >> half_lg, t = (e & half_mask) << 1;
      const float4 v = *reinterpret_cast<const float4*>(tile + perm_swz((j << lg) + t));
      const int64_t off = base_d[buf][j] + t_dst[t];
      if (p.mode == 0) {
        __stcs(reinterpret_cast<float4*>(static_cast<float2*>(p.dst) + off), v);
      } else {
        const float ar = tf32_hi(v.x);
        const float ai = tf32_hi(v.y);
        const float br = tf32_hi(v.z);
        const float bi = tf32_hi(v.w);
        *reinterpret_cast<float2*>(d + off) = make_float2(ar, br);
        *reinterpret_cast<float2*>(d + off + 2 * p.plane_stride) = make_float2(ai, bi);
        if (p.mode >= 3) {
          store_mix_x(d + p.plane_stride, off, v.x, p.mode == 4);
          store_mix_x(d + p.plane_stride, off + 1, v.z, p.mode == 4);
          store_mix_x(d + 3 * p.plane_stride, off, v.y, p.mode == 4);
          store_mix_x(d + 3 * p.plane_stride, off + 1, v.w, p.mode == 4);
        } else {
          const float ail = tf32_lo(v.y, ai), bil = tf32_lo(v.w, bi);
          *reinterpret_cast<float2*>(d + off + p.plane_stride) = make_float2(tf32_lo(v.x, ar), tf32_lo(v.z, br));
          *reinterpret_cast<float2*>(d + off + 3 * p.plane_stride) = make_float2(ail, bil);
          if (p.mode == 2) {  // stacked-B operand: negated imaginary planes
            *reinterpret_cast<float2*>(d + off + 4 * p.plane_stride) = make_float2(-ai, -bi);
            *reinterpret_cast<float2*>(d + off + 5 * p.plane_stride) = make_float2(-ail, -bil);
          }
        }
      }
    }
    if (!more) break;
    __syncthreads();
    c = cn;
    buf ^= 1;
  }
  if constexpr (DOT) perm_dot_reduce(dre, dim, p.partial);
}

cudaError_t launch_perm(const PermParams& p, cudaStream_t st) {
  const size_t smem = (((size_t)3 * p.ts * 4 + 15) & ~(size_t)15) + (size_t)p.ts * p.group * 8;
  const int64_t nchunks = (p.n_outer + p.group - 1) / p.group;
  int blocks = (int)std::min<int64_t>(nchunks, 148 * 8);
  if (blocks < 1) blocks = 1;
  if (p.vec && p.ts * p.group <= 2048) {
    static bool carveout = [] {
      cudaFuncSetAttribute(perm_vec_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      cudaFuncSetAttribute(perm_vec_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      return true;
    }();
    (void)carveout;
    if (p.mode == 5)
      launch_pdl(perm_vec_kernel<true>, blocks, 256, smem, st, p);
    else
      launch_pdl(perm_vec_kernel<false>, blocks, 256, smem, st, p);
  }
  else
    launch_pdl(perm_kernel, blocks, 256, smem, st, p);
  return cudaGetLastError();
}

cudaError_t launch_perm_dot(PermParams p, float2* partial, float2* z, cudaStream_t st) {
  p.mode = 5;
  p.partial = partial;
  const int64_t nchunks = (p.n_outer + p.group - 1) / p.group;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(nchunks, 148 * 8));
  cudaError_t e = launch_perm(p, st);
  if (e != cudaSuccess) return e;
  launch_pdl(simt_finalize_kernel, 1, 128, 0, st, partial, z, 1, blocks);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ dot
__global__ void __launch_bounds__(256) dot_kernel(const DotParams p) {
  pdl_wait();
  const int64_t n2 = p.n >> 1;  // complex pairs (16 B)
  const float4* x4 = reinterpret_cast<const float4*>(p.x);
  const float4* y4 = reinterpret_cast<const float4*>(p.y);
  float re = 0.f, im = 0.f, re2 = 0.f, im2 = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto mac = [](const float4 a, const float4 b, float& r, float& m) {
    r = fmaf(a.x, b.x, r);
    r = fmaf(-a.y, b.y, r);
    m = fmaf(a.x, b.y, m);
    m = fmaf(a.y, b.x, m);
    r = fmaf(a.z, b.z, r);
    r = fmaf(-a.w, b.w, r);
    m = fmaf(a.z, b.w, m);
    m = fmaf(a.w, b.z, m);
  };
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n2; i += 2 * stride) {  // two independent 32-byte load pairs in flight
    const float4 a0 = __ldcs(x4 + i), b0 = __ldcs(y4 + i);
    const float4 a1 = __ldcs(x4 + i + stride), b1 = __ldcs(y4 + i + stride);
    mac(a0, b0, re, im);
    mac(a1, b1, re2, im2);
  }
  if (i < n2) mac(__ldcs(x4 + i), __ldcs(y4 + i), re, im);
  re += re2;
  im += im2;
  if ((p.n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const float2 a = p.x[p.n - 1], b = p.y[p.n - 1];
    re += a.x * b.x - a.y * b.y;
    im += a.x * b.y + a.y * b.x;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, off);
    im += __shfl_xor_sync(0xffffffffu, im, off);
  }
  __shared__ float2 red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = make_float2(re, im);
  __syncthreads();
  if (threadIdx.x == 0) {
    float2 v = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      v.x += red[w].x;
      v.y += red[w].y;
    }
    p.partial[blockIdx.x] = v;
  }
}

cudaError_t launch_dot(const DotParams& p, cudaStream_t st) {
  launch_pdl(dot_kernel, p.nblocks, 256, 0, st, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  launch_pdl(simt_finalize_kernel, 1, 128, 0, st, p.partial, p.z, 1, p.nblocks);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ accumulate
__global__ void accum_kernel(const AccumParams p) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t o = tid; o < p.out_size; o += stride) {
    int64_t off = 0;
    decode1(p.out, o, off);
    double re = 0.0, im = 0.0;
    for (int64_t e = 0; e < p.extra_size; ++e) {
      int64_t eo = off;
      decode1(p.extra, e, eo);
      float2 v = p.root[eo];
      re += v.x;
      im += v.y;
    }
    if (p.acc_exp) {
      // exponent-tracking accumulation: acc[o] * 2^acc_exp[o] += (re, im) * 2^e
      const long long e = *p.hoist_exp + *p.slice_exp;
      double2 s = p.acc[o];
      long long ae = p.acc_exp[o];
      if (re != 0.0 || im != 0.0) {
        if (s.x == 0.0 && s.y == 0.0) {
          s = make_double2(re, im);
          ae = e;
        } else if (e > ae) {
          const double f = ldexp(1.0, (int)max(-1100LL, ae - e));
          s = make_double2(s.x * f + re, s.y * f + im);
          ae = e;
        } else {
          const double f = ldexp(1.0, (int)max(-1100LL, e - ae));
          s = make_double2(s.x + re * f, s.y + im * f);
        }
      }
      p.acc[o] = s;
      p.acc_exp[o] = ae;
      continue;
    }
    // Kahan-compensated complex128 accumulation
    double2 s = p.acc[o], c = p.comp[o];
    double yr = re - c.x, yi = im - c.y;
    double tr = s.x + yr, ti = s.y + yi;
    c.x = (tr - s.x) - yr;
    c.y = (ti - s.y) - yi;
    p.acc[o] = make_double2(tr, ti);
    p.comp[o] = c;
  }
  if (tid == 0 && p.slice_counter) *p.slice_counter += 1ull;
}

cudaError_t launch_accum(const AccumParams& p, cudaStream_t st) {
  launch_pdl(accum_kernel, grid_for(p.out_size, 256, 148 * 8), 256, 0, st, p);
  return cudaGetLastError();
}

// All-reduce of n plans' accumulators gathered into one buffer ([n][out]):
// Kahan sum of (acc_i - comp_i) (SPEC.md:551 compensated, order-fixed), or in
// strip_exponent mode the exponent-aligned sum of acc_i * 2^exp_i.
__global__ void allreduce_kernel(const double2* __restrict__ acc, const double2* __restrict__ comp,
                                 const long long* __restrict__ exps, int n, int64_t out_size,
                                 double2* out_acc, double2* out_comp, long long* out_exp) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < out_size; o += stride) {
    if (exps) {
      long long emax = LLONG_MIN;
      for (int i = 0; i < n; ++i) {
        const double2 v = acc[i * out_size + o];
        if (v.x != 0.0 || v.y != 0.0) emax = max(emax, exps[i * out_size + o]);
      }
      double2 s = make_double2(0.0, 0.0);
      if (emax != LLONG_MIN) {
        for (int i = 0; i < n; ++i) {
          const double2 v = acc[i * out_size + o];
          if (v.x == 0.0 && v.y == 0.0) continue;
          const double f = ldexp(1.0, (int)max(-1100LL, exps[i * out_size + o] - emax));
          s.x += v.x * f;
          s.y += v.y * f;
        }
      }
      out_acc[o] = s;
      out_exp[o] = emax == LLONG_MIN ? 0 : emax;
      continue;
    }
    double2 s = make_double2(0.0, 0.0), c = make_double2(0.0, 0.0);
    for (int t = 0; t < 2 * n; ++t) {
      const int i = t >> 1;
      double2 x = (t & 1) ? comp[i * out_size + o] : acc[i * out_size + o];
      if (t & 1) x = make_double2(-x.x, -x.y);
      const double yr = x.x - c.x, yi = x.y - c.y;
      const double tr = s.x + yr, ti = s.y + yi;
      c.x = (tr - s.x) - yr;
      c.y = (ti - s.y) - yi;
      s = make_double2(tr, ti);
    }
    out_acc[o] = s;
    out_comp[o] = c;
  }
}

cudaError_t launch_allreduce(const double2* acc, const double2* comp, const long long* exps, int n,
                             int64_t out_size, double2* out_acc, double2* out_comp, long long* out_exp,
                             cudaStream_t st) {
  launch_pdl(allreduce_kernel, grid_for(out_size, 256, 148 * 8), 256, 0, st, acc, comp, exps, n, out_size, out_acc,
                                                                    out_comp, out_exp);
  return cudaGetLastError();
}

__global__ void absmax_kernel(const float2* __restrict__ z, int64_t n, unsigned int* bits) {
  pdl_wait();
  float m = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float2 v = z[i];
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(bits, __float_as_uint(m));
}

__global__ void rescale_kernel(float2* __restrict__ z, int64_t n, const unsigned int* bits,
                               long long* exp_acc) {
  pdl_wait();
  const float m = __uint_as_float(*bits);
  if (!(m > 0.f) || !isfinite(m)) return;
  int e;
  frexpf(m, &e);  // m = f * 2^e, f in [0.5, 1)
  if (e == 0) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float2 v = z[i];
    z[i] = make_float2(ldexpf(v.x, -e), ldexpf(v.y, -e));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd((unsigned long long*)exp_acc, (unsigned long long)(long long)e);
}

cudaError_t launch_absmax(const float2* z, int64_t n, unsigned int* bits, cudaStream_t st) {
  launch_pdl(absmax_kernel, grid_for(n, 256, 148 * 8), 256, 0, st, z, n, bits);
  return cudaGetLastError();
}

cudaError_t launch_rescale(float2* z, int64_t n, const unsigned int* bits, long long* exp_acc,
                           cudaStream_t st) {
  launch_pdl(rescale_kernel, grid_for(n, 256, 148 * 8), 256, 0, st, z, n, bits, exp_acc);
  return cudaGetLastError();
}

__global__ void set_counter_kernel(unsigned long long* c, unsigned long long v) {
  pdl_wait(); *c = v; }

cudaError_t launch_set_counter(unsigned long long* counter, unsigned long long v, cudaStream_t st) {
  launch_pdl(set_counter_kernel, 1, 1, 0, st, counter, v);
  return cudaGetLastError();
}

// Clock stamps for measurement: every block records (SM id, clock64,
// globaltimer).  Two stamps bracketing a timed region give each SM's cycle
// count over the region and hence the mean SM clock it ran at.
__global__ void clock_stamp_kernel(unsigned long long* out) {
  if (threadIdx.x != 0) return;
  unsigned int smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  unsigned long long gt;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
  out[3 * blockIdx.x] = smid;
  out[3 * blockIdx.x + 1] = clock64();
  out[3 * blockIdx.x + 2] = gt;
}

cudaError_t launch_clock_stamp(unsigned long long* out, int blocks, cudaStream_t st) {
  clock_stamp_kernel<<<blocks, 32, 0, st>>>(out);
  return cudaGetLastError();
}

__global__ void convert_kernel(const double2* __restrict__ s, float2* __restrict__ d, int64_t n) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    d[i] = make_float2((float)s[i].x, (float)s[i].y);
}

cudaError_t launch_convert_c128(const double2* src, float2* dst, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  launch_pdl(convert_kernel, grid_for(n, 256, 148 * 8), 256, 0, st, src, dst, n);
  return cudaGetLastError();
}

cudaError_t launch_zero(void* p, int64_t bytes, cudaStream_t st) {
  return cudaMemsetAsync(p, 0, (size_t)bytes, st);
}

}  // namespace tnx
