// libtnx: plan compiler, HBM arena planner and per-slice runtime of the B200
// sliced contraction-tree executor.  C ABI in include/tnx.h.
//
// Reference semantics restated here (all citations /root/reference/...):
//   * appearances = #carrier leaves + 1 if output   hypergraph.py:39-57
//   * keep set of vertex v: labels whose accumulated leaf count is below the
//     appearance count; order = survivors of a, then b's new labels
//                                                   hypergraph.py:106-119,
//                                                   tree.py:137-169
//   * MACs per vertex = prod dims(s_a U s_b)        hypergraph.py:121-131
//   * W = log2 max internal result size, C = sum    tree.py:172-190
//   * slicing: sliced labels deleted from every incidence set, leaves
//     projected with fix_index                      SPEC.md:463-482, dense.py:161-170
//   * per pair: shared&kept = batch, shared&!kept = contracted,
//     exclusive&!kept = single-operand sum          dense.py:61-76
//   * slice ids: mixed radix over the SliceSet order, last label fastest
//                                                   SURVEY.md §8(a) a14
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "tnx.h"
#include "tnx_kernels.h"

using namespace tnx;
typedef unsigned __int128 u128;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// TNX_SIMT_PLANES=0 disables the SIMT -> GEMM operand-plane fusion (A/B)
static bool simt_planes_off() {
  static const int v = getenv("TNX_SIMT_PLANES") ? atoi(getenv("TNX_SIMT_PLANES")) : 1;
  return v == 0;
}

// TNX_GEMM_DPAIR=0 disables the paired full-line direct-plane stores (A/B)
static bool dpair_off() {
  static const int v = getenv("TNX_GEMM_DPAIR") ? atoi(getenv("TNX_GEMM_DPAIR")) : 1;
  return v == 0;
}

#define TNX_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t e__ = (call);                                                           \
    if (e__ != cudaSuccess)                                                             \
      return fail(TNX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__));   \
  } while (0)

namespace {

constexpr int64_t kAlign = 256;
inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Block {
  int64_t bytes = 0;
  int first = 0, last = 0;
  int64_t offset = 0;
};

// Greedy-by-size interval packing: largest blocks first, each placed at the
// lowest offset that does not overlap a time-overlapping placed block.
int64_t pack_blocks(std::vector<Block>& blocks) {
  std::vector<int> order(blocks.size());
  for (size_t i = 0; i < blocks.size(); ++i) order[i] = (int)i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return blocks[a].bytes > blocks[b].bytes; });
  std::vector<int> placed;
  int64_t total = 0;
  for (int i : order) {
    Block& bl = blocks[i];
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (int j : placed) {
      const Block& o = blocks[j];
      if (o.last < bl.first || bl.last < o.first) continue;
      busy.push_back({o.offset, o.offset + o.bytes});
    }
    std::sort(busy.begin(), busy.end());
    int64_t off = 0;
    for (auto& iv : busy) {
      if (off + bl.bytes <= iv.first) break;
      off = std::max(off, align_up(iv.second, kAlign));
    }
    bl.offset = off;
    total = std::max(total, off + bl.bytes);
    placed.push_back(i);
  }
  return align_up(total, kAlign);
}

enum Arena { AR_POOL = 0, AR_PERSIST = 1, AR_WORK = 2 };

struct TensorLoc {
  std::vector<int> labels;   // memory layout, row-major (last fastest)
  int64_t size = 1;
  int arena = AR_WORK;
  int phase = 1;             // 0 hoist, 1 slice (work arena blocks)
  int block = -1;
  int64_t offset = 0;        // pool: element offset; persist: byte offset
  bool fused = false;        // never materialised (written as parent operand planes)
};

enum VKind { VK_SIMT_T = 0, VK_SIMT_W = 1, VK_SIMT_S = 2, VK_GEMM = 3, VK_DOT = 4 };

struct Vertex {
  int ssa = 0, a = 0, b = 0;
  bool dep = false, hoisted = false;
  int kind = VK_SIMT_T;
  u128 macs = 0;
  std::vector<int> bl, cl, ml, nl, dxl, dyl;
  int64_t B = 1, M = 1, N = 1, K = 1, kp = 0, sum_size = 1;
  int nsplit = 0;
  int64_t chunk = 0;
  int blk_apl = -1, blk_bpl = -1, blk_part = -1, blk_tmp = -1;
  int splits = 1;
  int two_sm = 0;                   // 2-CTA GEMM configuration
  bool stack = false;               // stacked-B variant (B planes carry -im_hi, -im_lo)
  bool swap = false;  // GEMM A operand taken from y (larger row count)
  int plane_parent = -1;            // batched SIMT writes the parent GEMM's operand planes
  int plane_side = -1;
  int direct_parent = -1;           // GEMM writes the parent's operand planes
  int direct_side = -1;
  bool side_direct[2] = {false, false};  // operand planes written by a child GEMM
  int64_t tab_off = -1;  // element offset in the sum-table buffer
};

enum LaunchType { L_GATHER, L_SIMT, L_PACK, L_GEMM, L_ACCUM, L_PERM, L_DOT, L_SIMTB, L_RENORM, L_RESET };
struct Launch {
  int type;
  int idx;
  int vertex;  // ssa id or -1
};

struct Plan {
  int device = 0, precision = 1;
  uint32_t flags = 0;
  double gemm_min_macs = 0;
  int L = 0, n = 0;
  std::vector<int64_t> dims;
  std::vector<std::vector<int>> leaf_labels;
  std::vector<std::pair<int, int>> pairs;
  std::vector<int> output, sliced;
  std::vector<int> slice_pos;  // label -> position in sliced or -1
  u128 d = 1;
  std::vector<std::vector<std::pair<int, int>>> terms;
  std::vector<int> parent;
  std::vector<char> dep;
  std::vector<TensorLoc> T;
  std::vector<Vertex> V;  // index k <-> ssa n+k
  std::vector<int> hoist_order, slice_order;
  std::vector<int> gather_leaves;
  std::vector<int64_t> pool_off;
  int64_t pool_elems = 0;
  std::vector<Block> blocks[2];
  int64_t work_bytes = 0, persist_bytes = 0;
  u128 ops = 0;
  double width = 0;
  u128 peak = 0;
  int64_t out_size = 1;
  bool too_wide = false;
  std::vector<Int2Off> tables;
  std::vector<int32_t> ptabs;   // tiled-permutation tables
  int32_t* d_ptabs = nullptr;
  int64_t max_partial = 0;

  // device state
  bool bound = false;
  float2* pool = nullptr;
  char* work = nullptr;
  char* persist = nullptr;
  float2* partial = nullptr;
  Int2Off* d_tabs = nullptr;
  GatherJob* d_jobs = nullptr;
  int32_t* d_gstart = nullptr;
  void* ar_buf = nullptr;      // tnx_allreduce gather buffer (root plan)
  int64_t ar_bytes = 0;
  int njobs = 0;
  int gather_blocks = 0;
  double2* acc = nullptr;
  double2* comp = nullptr;
  unsigned long long* counter = nullptr;
  cudaStream_t own = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraph_t hgraph = nullptr;       // hoisted phase (replayed by every re-bind)
  cudaGraphExec_t hgexec = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::vector<Launch> hoist_launches, slice_launches;
  std::vector<SimtParams> simt;
  std::vector<PackParams> packs;
  std::vector<PermParams> perms;
  std::vector<DotParams> dots;
  struct SimtBatch {
    int64_t job_off = 0, start_off = 0;
    int njobs = 0, total_blocks = 0;
    std::vector<int> vertices;
  };
  std::vector<SimtBatch> batches;
  std::vector<SimtParams> bjobs;   // all batched jobs (device copy d_bjobs)
  std::vector<int32_t> bstarts;    // per batch: njobs + 1 block prefixes
  SimtParams* d_bjobs = nullptr;
  int32_t* d_bstarts = nullptr;
  // strip_exponent scratch: per-vertex abs-max bits, exponent counters
  unsigned int* d_absmax = nullptr;
  long long* d_exps = nullptr;     // [0] hoist exponent, [1] slice exponent
  long long* d_acc_exp = nullptr;
  bool strip() const { return (flags & TNX_FLAG_STRIP_EXPONENT) != 0; }
  std::vector<int> level;          // slice-phase dependency level per vertex index
  std::vector<GemmPlan> gemms;
  AccumParams accum{};
  float2* staging = nullptr;       // pinned host staging for complex128 leaf uploads
  // cross-stream ordering: every call that enqueues work records `order_ev` on
  // its stream; a later call on another stream waits on it first (bind / run /
  // reset / result share the arena, the accumulator and the staging buffer)
  cudaEvent_t order_ev = nullptr;
  cudaStream_t last_stream = nullptr;
  bool order_valid = false;

  ~Plan() { release(); }
  void release() {
    if (order_ev) cudaEventDestroy(order_ev);
    order_ev = nullptr;
    order_valid = false;
    if (gexec) cudaGraphExecDestroy(gexec);
    if (graph) cudaGraphDestroy(graph);
    if (hgexec) cudaGraphExecDestroy(hgexec);
    if (hgraph) cudaGraphDestroy(hgraph);
    gexec = nullptr;
    graph = nullptr;
    hgexec = nullptr;
    hgraph = nullptr;
    void* ptrs[] = {pool,    work,   persist, partial, d_tabs,    d_jobs,   acc,    comp,
                    counter, d_ptabs, d_bjobs, d_bstarts, d_absmax, d_exps, d_acc_exp, d_gstart, ar_buf};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    pool = nullptr;
    work = persist = nullptr;
    partial = nullptr;
    d_tabs = nullptr;
    d_ptabs = nullptr;
    d_bjobs = nullptr;
    d_bstarts = nullptr;
    d_absmax = nullptr;
    d_exps = nullptr;
    d_acc_exp = nullptr;
    d_jobs = nullptr;
    d_gstart = nullptr;
    ar_buf = nullptr;
    ar_bytes = 0;
    acc = comp = nullptr;
    counter = nullptr;
    if (own) cudaStreamDestroy(own);
    own = nullptr;
    if (staging) cudaFreeHost(staging);
    staging = nullptr;
    bound = false;
  }

  int64_t prod(const std::vector<int>& ls) const {
    int64_t p = 1;
    for (int l : ls) p *= dims[l];
    return p;
  }
  int64_t stride_in(const TensorLoc& t, int label) const {
    int64_t s = 1;
    for (int i = (int)t.labels.size() - 1; i >= 0; --i) {
      if (t.labels[i] == label) return s;
      s *= dims[t.labels[i]];
    }
    return 0;
  }
  float2* ptr(const TensorLoc& t) const {
    if (t.arena == AR_POOL) return pool + t.offset;
    if (t.arena == AR_PERSIST) return reinterpret_cast<float2*>(persist + t.offset);
    return reinterpret_cast<float2*>(work + blocks[t.phase][t.block].offset);
  }
  char* block_ptr(int phase, int blk) const { return work + blocks[phase][blk].offset; }
};

// Build a fused IdxMap over `labels` (iteration order, last fastest) with the
// strides of up to two tensors (stride 0 when a label is absent).
bool build_map(const Plan& P, const std::vector<int>& labels, const TensorLoc* t0,
               const TensorLoc* t1, IdxMap& m, std::string& err) {
  std::vector<int64_t> dm, s0, s1;
  for (int l : labels) {
    int64_t d = P.dims[l];
    int64_t a = t0 ? P.stride_in(*t0, l) : 0;
    int64_t b = t1 ? P.stride_in(*t1, l) : 0;
    if (d == 1) continue;
    if (!dm.empty() && s0.back() == a * d && s1.back() == b * d) {
      dm.back() *= d;
      s0.back() = a;
      s1.back() = b;
      continue;
    }
    dm.push_back(d);
    s0.push_back(a);
    s1.push_back(b);
  }
  std::memset(&m, 0, sizeof(m));
  if ((int)dm.size() > kMaxGroups) {
    err = "index map needs " + std::to_string(dm.size()) + " groups (max " +
          std::to_string(kMaxGroups) + ")";
    return false;
  }
  m.n = (int)dm.size();
  for (int i = 0; i < m.n; ++i) {
    m.dim[i] = dm[i];
    m.st0[i] = s0[i];
    m.st1[i] = s1[i];
    int lg = -1;
    if ((dm[i] & (dm[i] - 1)) == 0) {
      lg = 0;
      while ((int64_t(1) << lg) < dm[i]) ++lg;
    }
    m.lg[i] = (int8_t)lg;
  }
  return true;
}

// Label order of the K-blocked operand planes of GEMM vertex v, side 0 (A)
// or 1 (B): row-major [K outer][batch + side rows][K inner, product 16].
// False when K is padded or no K suffix has product 16 (gather-pack path).
bool plane_order(const Plan& P, const Vertex& v, int side, std::vector<int>& dst) {
  if (v.kp != v.K) return false;
  int64_t pr = 1;
  int i = (int)v.cl.size() - 1;
  for (; i >= 0 && pr < 16; --i) pr *= P.dims[v.cl[i]];
  if (pr != 16) return false;
  const std::vector<int>& own = (side == 0) != v.swap ? v.ml : v.nl;
  dst.assign(v.cl.begin(), v.cl.begin() + (i + 1));
  dst.insert(dst.end(), v.bl.begin(), v.bl.end());
  dst.insert(dst.end(), own.begin(), own.end());
  dst.insert(dst.end(), v.cl.begin() + (i + 1), v.cl.end());
  return true;
}

int compile(Plan& P, const tnx_plan_desc* D) {
  P.L = D->num_labels;
  P.n = D->num_leaves;
  P.device = D->device;
  P.precision = D->precision;
  P.flags = D->flags;
  P.gemm_min_macs = D->gemm_min_macs > 0 ? D->gemm_min_macs : double(1 << 22);
  if (P.L < 0 || P.n < 1) return fail(TNX_ERR_INVALID, "empty tree");
  P.dims.assign(D->label_dims, D->label_dims + P.L);
  for (int l = 0; l < P.L; ++l)
    if (P.dims[l] < 1) return fail(TNX_ERR_DATA, "index " + std::to_string(l) + " has non-positive dim");
  // leaves
  int64_t pos = 0;
  P.leaf_labels.resize(P.n);
  std::vector<int> app(P.L, 0);
  for (int i = 0; i < P.n; ++i) {
    int r = D->leaf_ranks[i];
    if (r < 0) return fail(TNX_ERR_DATA, "negative leaf rank");
    std::vector<int>& ls = P.leaf_labels[i];
    for (int j = 0; j < r; ++j) {
      int l = D->leaf_labels[pos + j];
      if (l < 0 || l >= P.L) return fail(TNX_ERR_DATA, "unknown index id in leaf " + std::to_string(i));
      if (std::find(ls.begin(), ls.end(), l) != ls.end())
        return fail(TNX_ERR_DATA, "repeated index in leaf " + std::to_string(i));
      ls.push_back(l);
      app[l] += 1;
    }
    pos += r;
  }
  for (int j = 0; j < D->num_output; ++j) {
    int l = D->output_labels[j];
    if (l < 0 || l >= P.L) return fail(TNX_ERR_DATA, "unknown output index");
    if (app[l] == 0) return fail(TNX_ERR_DATA, "output index appears in no node");
    if (std::find(P.output.begin(), P.output.end(), l) != P.output.end())
      return fail(TNX_ERR_DATA, "repeated output index");
    P.output.push_back(l);
  }
  for (int l : P.output) app[l] += 1;
  P.slice_pos.assign(P.L, -1);
  for (int j = 0; j < D->num_sliced; ++j) {
    int l = D->sliced_labels[j];
    if (l < 0 || l >= P.L) return fail(TNX_ERR_INVALID, "unknown sliced label");
    if (P.slice_pos[l] >= 0) return fail(TNX_ERR_INVALID, "repeated label in slice set");
    if (std::find(P.output.begin(), P.output.end(), l) != P.output.end())
      return fail(TNX_ERR_INVALID, "output label cannot be sliced");
    P.slice_pos[l] = (int)P.sliced.size();
    P.sliced.push_back(l);
    P.d *= (u128)P.dims[l];
  }
  if (P.d > (u128)(~0ull >> 1)) return fail(TNX_ERR_INVALID, "d_sliced exceeds 2^63");
  // tree validation (tree.py:43-56)
  const int nv = P.n > 1 ? 2 * P.n - 1 : 1;
  P.pairs.resize(P.n - 1);
  P.parent.assign(nv, -1);
  for (int k = 0; k < P.n - 1; ++k) {
    int a = D->pairs[2 * k], b = D->pairs[2 * k + 1];
    for (int c : {a, b}) {
      if (c < 0 || c >= P.n + k)
        return fail(TNX_ERR_INVALID, "pair " + std::to_string(k) + " references unbuilt vertex " + std::to_string(c));
      if (P.parent[c] >= 0) return fail(TNX_ERR_INVALID, "vertex " + std::to_string(c) + " consumed twice");
      P.parent[c] = P.n + k;
    }
    if (a == b) return fail(TNX_ERR_INVALID, "vertex consumed twice");
    P.pairs[k] = {a, b};
  }
  // terms (label-count saturation)
  P.terms.resize(nv);
  for (int i = 0; i < P.n; ++i)
    for (int l : P.leaf_labels[i]) P.terms[i].push_back({l, 1});
  std::vector<int> cnt(P.L, 0), seen(P.L, -1);
  for (int k = 0; k < P.n - 1; ++k) {
    const auto& ta = P.terms[P.pairs[k].first];
    const auto& tb = P.terms[P.pairs[k].second];
    auto& out = P.terms[P.n + k];
    for (auto& e : tb) {
      cnt[e.first] = e.second;
      seen[e.first] = k;
    }
    for (auto& e : ta) {
      int c = e.second + (seen[e.first] == k ? cnt[e.first] : 0);
      if (c < app[e.first]) out.push_back({e.first, c});
    }
    for (auto& e : ta) seen[e.first] = -2 - k;  // mark as present in a
    for (auto& e : tb) {
      if (seen[e.first] == -2 - k) continue;
      if (e.second < app[e.first]) out.push_back({e.first, e.second});
    }
  }
  // dependence on sliced labels
  P.dep.assign(nv, 0);
  for (int i = 0; i < P.n; ++i)
    for (int l : P.leaf_labels[i])
      if (P.slice_pos[l] >= 0) P.dep[i] = 1;
  for (int k = 0; k < P.n - 1; ++k)
    P.dep[P.n + k] = P.dep[P.pairs[k].first] | P.dep[P.pairs[k].second];
  const bool hoist = P.d > 1 && !(P.flags & TNX_FLAG_NO_HOIST);

  // leaf pool + leaf tensors
  P.T.resize(nv);
  P.pool_off.resize(P.n);
  int64_t poff = 0;
  for (int i = 0; i < P.n; ++i) {
    int64_t sz = 1;
    for (int l : P.leaf_labels[i]) sz *= P.dims[l];
    P.pool_off[i] = poff;
    poff += align_up(sz, 32);
  }
  P.pool_elems = std::max<int64_t>(poff, 32);
  for (int i = 0; i < P.n; ++i) {
    TensorLoc& t = P.T[i];
    bool sl = false;
    for (int l : P.leaf_labels[i]) {
      if (P.slice_pos[l] >= 0) sl = true;
      else t.labels.push_back(l);
    }
    t.size = P.prod(t.labels);
    if (!sl) {
      t.arena = AR_POOL;
      t.offset = P.pool_off[i];
    } else {
      t.arena = AR_WORK;
      t.phase = 1;
      P.gather_leaves.push_back(i);
    }
  }
  // bookkeeping: ops, width
  P.V.resize(P.n - 1);
  P.peak = 0;
  for (int k = 0; k < P.n - 1; ++k) {
    Vertex& v = P.V[k];
    v.ssa = P.n + k;
    v.a = P.pairs[k].first;
    v.b = P.pairs[k].second;
    v.dep = P.dep[v.ssa];
    v.hoisted = hoist && !v.dep;
    u128 m = 1;
    std::vector<char> mark(P.L, 0);
    for (auto& e : P.terms[v.a]) mark[e.first] = 1;
    for (auto& e : P.terms[v.b]) mark[e.first] = 1;
    for (int l = 0; l < P.L; ++l)
      if (mark[l] && P.slice_pos[l] < 0) m *= (u128)P.dims[l];
    v.macs = m;
    P.ops += m;
    u128 sz = 1;
    for (auto& e : P.terms[v.ssa])
      if (P.slice_pos[e.first] < 0) sz *= (u128)P.dims[e.first];
    P.peak = std::max(P.peak, sz);
  }
  for (int l : P.output) P.out_size *= P.dims[l];
  if (P.n == 1) P.peak = (u128)P.out_size;
  P.width = (double)std::log2((long double)P.peak);
  // bookkeeping is exact at any width; lowering only for executable widths
  if (P.peak >= ((u128)1 << 40)) {
    P.too_wide = true;
    return TNX_OK;
  }

  // execution order: hoisted vertices in SSA order; slice-dependent vertices
  // by dependency level (all vertices of a level form one step: independent,
  // batched into shared launches, and disjoint in memory by construction)
  // (the hoisted phase is level-scheduled the same way within its own DAG)
  P.level.assign(P.n - 1, 0);
  for (int k = 0; k < P.n - 1; ++k) {
    int lv = 0;
    for (int c : {P.V[k].a, P.V[k].b})
      if (c >= P.n && P.V[c - P.n].hoisted == P.V[k].hoisted) lv = std::max(lv, P.level[c - P.n]);
    P.level[k] = lv + 1;
    (P.V[k].hoisted ? P.hoist_order : P.slice_order).push_back(k);
  }
  auto by_level = [&](int a, int b) { return P.level[a] < P.level[b]; };
  std::stable_sort(P.hoist_order.begin(), P.hoist_order.end(), by_level);
  std::stable_sort(P.slice_order.begin(), P.slice_order.end(), by_level);

  // per-vertex lowering + memory blocks
  auto add_block = [&](int phase, int64_t bytes, int first, int last) {
    Block b;
    b.bytes = align_up(std::max<int64_t>(bytes, 16), kAlign);
    b.first = first;
    b.last = last;
    P.blocks[phase].push_back(b);
    return (int)P.blocks[phase].size() - 1;
  };
  // step index of each vertex within its phase (slice phase: gather = 0)
  std::vector<int> step(nv, 0);
  for (int k : P.hoist_order) step[P.n + k] = P.level[k] - 1;
  int max_level = 0;
  for (int k : P.slice_order) {
    step[P.n + k] = P.level[k];
    max_level = std::max(max_level, P.level[k]);
  }
  const int accum_step = max_level + 1;
  const int root = P.n > 1 ? 2 * P.n - 2 : 0;
  auto consumer_step = [&](int v) {
    int p = P.parent[v];
    if (p < 0) return accum_step;  // root
    return step[p];
  };
  for (int i : P.gather_leaves)
    P.T[i].block = add_block(1, P.T[i].size * 8, 0, consumer_step(i));

  int64_t persist_off = 0;
  for (int k = 0; k < P.n - 1; ++k) {
    Vertex& v = P.V[k];
    const TensorLoc& x = P.T[v.a];
    const TensorLoc& y = P.T[v.b];
    std::vector<char> inx(P.L, 0), iny(P.L, 0), keep(P.L, 0);
    for (int l : x.labels) inx[l] = 1;
    for (int l : y.labels) iny[l] = 1;
    for (auto& e : P.terms[v.ssa])
      if (P.slice_pos[e.first] < 0) keep[e.first] = 1;
    for (int l : x.labels) {
      if (iny[l]) (keep[l] ? v.bl : v.cl).push_back(l);
      else (keep[l] ? v.ml : v.dxl).push_back(l);
    }
    for (int l : y.labels)
      if (!inx[l]) (keep[l] ? v.nl : v.dyl).push_back(l);
    v.B = P.prod(v.bl);
    v.M = P.prod(v.ml);
    v.N = P.prod(v.nl);
    v.K = P.prod(v.cl);
    v.sum_size = v.K * P.prod(v.dxl) * P.prod(v.dyl);
    TensorLoc& z = P.T[v.ssa];
    // tensor cores for GEMM-shaped vertices; small K (padded to 16) still
    // goes there when the output is large (SIMT would be output-bound)
    // tcgen05 GEMM: K >= 16 contractions with enough MACs even for narrow M / N
    // (a 128-row tile at half utilisation beats the SIMT kernels by >10x; below 64
    // rows the extra TF32 error outweighs it -- a 7x7 amplitude test crossed 1e-5 at 16;
    // rows / columns past M / N are computed and masked), small-K ones only
    // when the output is large (SIMT would be output-bound)
    static const int64_t min_mn = getenv("TNX_GEMM_MIN_MN") ? atoll(getenv("TNX_GEMM_MIN_MN")) : 64;
    const bool gemm = P.precision != TNX_PREC_FP32 && v.dxl.empty() && v.dyl.empty() &&
                      (v.K >= 16 ? std::min(v.M, v.N) >= min_mn && (double)v.macs >= P.gemm_min_macs
                                 : v.M >= 128 && v.N >= 128 && v.M * v.N >= (int64_t(1) << 20));
    if (gemm) {
      v.kind = VK_GEMM;
      // A takes the operand with more rows (output rows = A rows)
      v.swap = v.N > v.M;
      z.labels = v.bl;
      const std::vector<int>& first = v.swap ? v.nl : v.ml;
      const std::vector<int>& second = v.swap ? v.ml : v.nl;
      z.labels.insert(z.labels.end(), first.begin(), first.end());
      z.labels.insert(z.labels.end(), second.begin(), second.end());
      v.kp = align_up(v.K, 16);
    } else {
      for (int l : x.labels)
        if (keep[l]) z.labels.push_back(l);
      for (int l : y.labels)
        if (keep[l] && !inx[l]) z.labels.push_back(l);
      const int64_t out = P.prod(z.labels);
      const int64_t par = 148 * 2048;
      if (out == 1 && v.dxl.empty() && v.dyl.empty() && v.bl.empty() && v.sum_size >= (1 << 16))
        v.kind = VK_DOT;  // full contraction: permute y to x's layout + streaming dot
      else if (v.sum_size <= 64 || out >= par / 2) v.kind = VK_SIMT_T;
      else if (out * 32 >= par / 2) v.kind = VK_SIMT_W;
      else {
        v.kind = VK_SIMT_S;
        int64_t ns = std::max<int64_t>(1, std::min<int64_t>((1184 + out - 1) / out, (v.sum_size + 2047) / 2048));
        v.nsplit = (int)ns;
        v.chunk = (v.sum_size + ns - 1) / ns;
        P.max_partial = std::max(P.max_partial, out * ns);
      }
    }
    z.size = P.prod(z.labels);
    // placement of the result
    const int ph = v.hoisted ? 0 : 1;
    const int st = step[v.ssa];
    const int par = P.parent[v.ssa];
    if (v.hoisted && (par < 0 || !P.V[par - P.n].hoisted)) {
      z.arena = AR_PERSIST;
      z.offset = persist_off;
      persist_off += align_up(z.size * 8, kAlign);
    } else {
      z.arena = AR_WORK;
      z.phase = ph;
      int last = v.hoisted ? (par >= 0 ? step[par] : st) : consumer_step(v.ssa);
      z.block = add_block(ph, z.size * 8, st, last);
    }
    if (v.kind == VK_DOT) {
      if (x.labels != y.labels) v.blk_tmp = add_block(ph, 8 * y.size, st, st);
      P.max_partial = std::max<int64_t>(P.max_partial, 148 * 8);  // dot / fused perm-dot block partials
    }
    if (v.kind == VK_GEMM) {
      const int64_t ra = v.swap ? v.N : v.M, rb = v.swap ? v.M : v.N;
      v.splits = ((v.B * v.M * v.N) % 2 == 0) ? gemm_choose_splits(v.B, ra, rb, v.kp) : 1;
      v.two_sm = gemm_use_2sm(v.B, ra, rb, v.kp, v.splits);
      v.stack = P.precision == TNX_PREC_3XTF32 && gemm_use_stack(v.B, ra, rb, v.kp, v.two_sm);
      v.blk_apl = add_block(ph, 16 * v.B * ra * v.kp, st, st);
      v.blk_bpl = add_block(ph, (v.stack ? 24 : 16) * v.B * rb * v.kp, st, st);
      if (v.splits > 1) v.blk_part = add_block(ph, 8 * (int64_t)v.splits * v.B * v.M * v.N, st, st);
    }
  }
  // GEMM -> GEMM fusion: a child GEMM writes its result straight into the
  // parent's split-TF32 operand planes (saves the parent's pack pass).  The
  // child's result is never materialised, so its orientation and row/column
  // label orders are free; decided top-down (root first) so every parent's
  // orientation is final before its children are arranged:
  //   * the parent's K order puts 4 labels (product 16) that sit on ONE side
  //     of the leading child innermost (they form the planes' 64 B K-inner run);
  //   * that child side becomes the child's row (A) side, and the child's rows
  //     and columns follow the parent's plane order, so the 32 lanes of an
  //     epilogue warp store consecutive floats (whole 128 B lines).
  if (P.precision != TNX_PREC_FP32 && !(P.flags & TNX_FLAG_NO_DIRECT) &&
      !(P.flags & TNX_FLAG_STRIP_EXPONENT)) {
    auto in_list = [](const std::vector<int>& v, int l) {
      return std::find(v.begin(), v.end(), l) != v.end();
    };
    auto refresh = [&](Vertex& v) {  // derived sizes after a swap / reorder
      const int ph = v.hoisted ? 0 : 1;
      const int64_t ra = v.swap ? v.N : v.M, rb = v.swap ? v.M : v.N;
      // the launch configuration follows the orientation (A rows pair up in 2-CTA mode)
      v.two_sm = gemm_use_2sm(v.B, ra, rb, v.kp, v.splits);
      v.stack = P.precision == TNX_PREC_3XTF32 && gemm_use_stack(v.B, ra, rb, v.kp, v.two_sm);
      P.blocks[ph][v.blk_apl].bytes = align_up(16 * v.B * ra * v.kp, kAlign);
      P.blocks[ph][v.blk_bpl].bytes = align_up((v.stack ? 24 : 16) * v.B * rb * v.kp, kAlign);
      TensorLoc& z = P.T[v.ssa];
      z.labels = v.bl;
      const std::vector<int>& f1 = v.swap ? v.nl : v.ml;
      const std::vector<int>& f2 = v.swap ? v.ml : v.nl;
      z.labels.insert(z.labels.end(), f1.begin(), f1.end());
      z.labels.insert(z.labels.end(), f2.begin(), f2.end());
    };
    for (int k = P.n - 2; k >= 0; --k) {
      Vertex& pv = P.V[k];
      if (pv.kind != VK_GEMM || pv.kp != pv.K) continue;
      int ch[2];
      bool cand[2];
      for (int side = 0; side < 2; ++side) {
        ch[side] = side == 0 ? (pv.swap ? pv.b : pv.a) : (pv.swap ? pv.a : pv.b);
        cand[side] = false;
        if (ch[side] < P.n) continue;
        const Vertex& cv = P.V[ch[side] - P.n];
        cand[side] = cv.kind == VK_GEMM && cv.splits == 1 && cv.hoisted == pv.hoisted;
      }
      if (!cand[0] && !cand[1]) continue;
      // K-inner labels: a product-16 run of parent K labels lying on ONE side
      // of each fused child (prefer a run that works for both children)
      const int lead = cand[0] ? 0 : 1;
      std::vector<int> kin;
      int side_of[2] = {-1, -1};  // per child: 0 = its ml side, 1 = its nl side
      auto pick16 = [&](const std::vector<int>& grp) {
        int64_t pr = 1;
        std::vector<int> pick;
        for (int i = (int)grp.size() - 1; i >= 0 && pr < 16; --i) {
          pr *= P.dims[grp[i]];
          pick.insert(pick.begin(), grp[i]);
        }
        return pr == 16 ? pick : std::vector<int>();
      };
      {
        int best = -1;
        for (int s0 = 0; s0 < 2; ++s0)
          for (int s1 = 0; s1 < (cand[0] && cand[1] ? 2 : 1); ++s1) {
            std::vector<int> grp;
            for (int l : pv.cl) {
              bool ok = true;
              for (int side = 0; side < 2; ++side) {
                if (!cand[side]) continue;
                const Vertex& cv = P.V[ch[side] - P.n];
                const int want = (side == lead) ? s0 : s1;
                ok = ok && in_list(want == 0 ? cv.ml : cv.nl, l);
              }
              if (ok) grp.push_back(l);
            }
            std::vector<int> pk = pick16(grp);
            if (!pk.empty() && (int)grp.size() > best) {
              best = (int)grp.size();
              kin = pk;
              side_of[lead] = s0;
              side_of[1 - lead] = s1;
            }
          }
        if (kin.empty()) {  // lead child only
          const Vertex& lc = P.V[ch[lead] - P.n];
          for (int s0 = 0; s0 < 2 && kin.empty(); ++s0) {
            std::vector<int> grp;
            for (int l : pv.cl)
              if (in_list(s0 == 0 ? lc.ml : lc.nl, l)) grp.push_back(l);
            kin = pick16(grp);
            if (!kin.empty()) side_of[lead] = s0;
          }
        }
      }
      if (!kin.empty()) {
        std::vector<int> ncl;
        for (int l : pv.cl)
          if (!in_list(kin, l)) ncl.push_back(l);
        ncl.insert(ncl.end(), kin.begin(), kin.end());
        pv.cl = ncl;
      }
      for (int side = 0; side < 2; ++side) {
        if (!cand[side]) continue;
        std::vector<int> dst;
        if (!plane_order(P, pv, side, dst)) continue;
        Vertex& cv = P.V[ch[side] - P.n];
        // orientation: the child side holding the K-inner run becomes its rows
        if (!kin.empty()) {
          bool all_m = true, all_n = true;
          for (int l : kin) {
            all_m = all_m && in_list(cv.ml, l);
            all_n = all_n && in_list(cv.nl, l);
          }
          if (side_of[side] == 0 && all_m) cv.swap = false;
          else if (side_of[side] == 1 && all_n) cv.swap = true;
          else if (all_m) cv.swap = false;
          else if (all_n) cv.swap = true;
        }
        std::vector<int64_t> pst(P.L, 0);
        int64_t acc = 1;
        for (int i = (int)dst.size() - 1; i >= 0; --i) {
          pst[dst[i]] = acc;
          acc *= P.dims[dst[i]];
        }
        auto by_stride = [&](int a, int b) { return pst[a] > pst[b]; };
        std::stable_sort(cv.ml.begin(), cv.ml.end(), by_stride);
        std::stable_sort(cv.nl.begin(), cv.nl.end(), by_stride);
        refresh(cv);
        cv.direct_parent = pv.ssa;
        cv.direct_side = side;
        pv.side_direct[side] = true;
        const int ph = pv.hoisted ? 0 : 1;
        Block& pb = P.blocks[ph][side == 0 ? pv.blk_apl : pv.blk_bpl];
        pb.first = std::min(pb.first, step[ch[side]]);
        TensorLoc& tc = P.T[ch[side]];
        if (tc.arena == AR_WORK && tc.block >= 0) P.blocks[ph][tc.block].bytes = kAlign;
        tc.fused = true;
      }
    }
  }
  // SIMT -> GEMM fusion: a small contraction (batched thread / warp mode) whose
  // parent is a GEMM writes its result straight into the parent's K-blocked
  // split-TF32 operand planes (no materialised tensor, no pack launch).  Its
  // output elements cover the planes exactly (K is not padded: plane_order).
  if (P.precision == TNX_PREC_3XTF32 && !(P.flags & TNX_FLAG_NO_DIRECT) &&
      !(P.flags & TNX_FLAG_STRIP_EXPONENT) && !simt_planes_off()) {
    for (int k = 0; k < P.n - 1; ++k) {
      Vertex& pv = P.V[k];
      if (pv.kind != VK_GEMM) continue;
      for (int side = 0; side < 2; ++side) {
        if (pv.side_direct[side]) continue;
        const int c = side == 0 ? (pv.swap ? pv.b : pv.a) : (pv.swap ? pv.a : pv.b);
        if (c < P.n) continue;
        Vertex& cv = P.V[c - P.n];
        if ((cv.kind != VK_SIMT_T && cv.kind != VK_SIMT_W) || cv.hoisted != pv.hoisted) continue;
        std::vector<int> dst;
        if (!plane_order(P, pv, side, dst)) continue;
        cv.plane_parent = pv.ssa;
        cv.plane_side = side;
        pv.side_direct[side] = true;
        const int ph = pv.hoisted ? 0 : 1;
        Block& pb = P.blocks[ph][side == 0 ? pv.blk_apl : pv.blk_bpl];
        pb.first = std::min(pb.first, step[c]);
        TensorLoc& tc = P.T[c];
        if (tc.arena == AR_WORK && tc.block >= 0) P.blocks[ph][tc.block].bytes = kAlign;
        tc.fused = true;
      }
    }
  }
  if (getenv("TNX_DEBUG_PLAN")) {
    for (auto& v : P.V) {
      if (v.kind != VK_GEMM) continue;
      std::string info;
      if (v.direct_parent >= 0) {
        const Vertex& pv = P.V[v.direct_parent - P.n];
        std::vector<int> dst;
        plane_order(P, pv, v.direct_side, dst);
        std::vector<int64_t> pst(P.L, 0);
        int64_t acc = 1;
        for (int i = (int)dst.size() - 1; i >= 0; --i) { pst[dst[i]] = acc; acc *= P.dims[dst[i]]; }
        const std::vector<int>& f1 = v.swap ? v.nl : v.ml;
        const std::vector<int>& f2 = v.swap ? v.ml : v.nl;
        info = " rows_inner_strides=";
        for (int i = std::max(0, (int)f1.size() - 6); i < (int)f1.size(); ++i) info += std::to_string(pst[f1[i]]) + ",";
        info += " cols_inner_strides=";
        for (int i = std::max(0, (int)f2.size() - 6); i < (int)f2.size(); ++i) info += std::to_string(pst[f2[i]]) + ",";
      }
      fprintf(stderr, "gemm v=%d M=%lld N=%lld K=%lld swap=%d splits=%d 2sm=%d stack=%d parent=%d side=%d%s\n",
              v.ssa, (long long)v.M, (long long)v.N, (long long)v.K, (int)v.swap, v.splits, v.two_sm,
              (int)v.stack, v.direct_parent, v.direct_side, info.c_str());
    }
  }
  P.persist_bytes = std::max<int64_t>(persist_off, kAlign);
  P.work_bytes = std::max(pack_blocks(P.blocks[0]), pack_blocks(P.blocks[1]));
  P.work_bytes = std::max<int64_t>(P.work_bytes, kAlign);
  (void)root;
  return TNX_OK;
}

// Tiled permutation of tensor t into the row-major order `dst` (same label
// set).  Tables are appended to P.ptabs (tab_off = element offset).  Returns
// false when the tile would be too large or offsets overflow int32.
bool build_perm(Plan& P, const TensorLoc& t, const std::vector<int>& dst, int mode,
                PermParams& pp, int64_t& tab_off, std::string& err) {
  std::memset(&pp, 0, sizeof(pp));
  if (t.size >= (int64_t(1) << 31)) return false;
  std::vector<char> in_tile(P.L, 0);
  static const int64_t run_src = getenv("TNX_PERM_SRC") ? atoll(getenv("TNX_PERM_SRC")) : 32;
  static const int64_t run_dst = getenv("TNX_PERM_DST") ? atoll(getenv("TNX_PERM_DST")) : 32;
  int64_t prod = 1;
  for (int i = (int)t.labels.size() - 1; i >= 0 && prod < run_src; --i) {
    prod *= P.dims[t.labels[i]];
    in_tile[t.labels[i]] = 1;
  }
  prod = 1;
  for (int i = (int)dst.size() - 1; i >= 0 && prod < run_dst; --i) {
    prod *= P.dims[dst[i]];
    in_tile[dst[i]] = 1;
  }
  std::vector<int> tsrc, tdst, outer;
  for (int l : t.labels)
    if (in_tile[l]) tsrc.push_back(l);
  for (int l : dst) (in_tile[l] ? tdst : outer).push_back(l);
  const int64_t ts = P.prod(tsrc);
  if (ts > 4096 || ts < 1) return false;
  // destination (row-major) strides
  std::vector<int64_t> dstr(P.L, 0);
  int64_t s = 1;
  for (int i = (int)dst.size() - 1; i >= 0; --i) {
    dstr[dst[i]] = s;
    s *= P.dims[dst[i]];
  }
  // strides within the dst-ordered tile
  std::vector<int64_t> tstr(P.L, 0);
  s = 1;
  for (int i = (int)tdst.size() - 1; i >= 0; --i) {
    tstr[tdst[i]] = s;
    s *= P.dims[tdst[i]];
  }
  tab_off = (int64_t)P.ptabs.size();
  P.ptabs.resize(P.ptabs.size() + 3 * ts);
  int32_t* T_src = P.ptabs.data() + tab_off;
  int32_t* T_idx = T_src + ts;
  int32_t* T_dst = T_idx + ts;
  auto walk = [&](const std::vector<int>& order, auto&& fn) {
    std::vector<int64_t> dig(order.size(), 0);
    for (int64_t e = 0; e < ts; ++e) {
      fn(e, dig);
      for (int i = (int)order.size() - 1; i >= 0; --i) {
        if (++dig[i] < P.dims[order[i]]) break;
        dig[i] = 0;
      }
    }
  };
  walk(tsrc, [&](int64_t e, const std::vector<int64_t>& dig) {
    int64_t so = 0, ti = 0;
    for (size_t i = 0; i < tsrc.size(); ++i) {
      so += dig[i] * P.stride_in(t, tsrc[i]);
      ti += dig[i] * tstr[tsrc[i]];
    }
    T_src[e] = (int32_t)so;
    T_idx[e] = (int32_t)ti;
  });
  walk(tdst, [&](int64_t e, const std::vector<int64_t>& dig) {
    int64_t d = 0;
    for (size_t i = 0; i < tdst.size(); ++i) d += dig[i] * dstr[tdst[i]];
    T_dst[e] = (int32_t)d;
  });
  // outer map: st0 = source stride, st1 = destination stride
  TensorLoc dl;
  dl.labels = dst;
  if (!build_map(P, outer, &t, &dl, pp.outer, err)) return false;
  pp.n_outer = P.prod(outer);
  pp.ts = (int32_t)ts;
  pp.group = (int32_t)std::max<int64_t>(1, std::min<int64_t>(64, 2048 / ts));
  pp.mode = mode;
  pp.ts_log2 = -1;
  if ((ts & (ts - 1)) == 0) {
    int lg = 0;
    while ((int64_t(1) << lg) < ts) ++lg;
    pp.ts_log2 = lg;
  }
  // vectorised path: pairs (t, t+1) contiguous and even-aligned on both sides,
  // outer strides even (so every base keeps the alignment)
  bool vec = pp.ts_log2 >= 1;
  for (int64_t e = 0; vec && e < ts; e += 2) {
    if (T_src[e + 1] != T_src[e] + 1 || (T_src[e] & 1)) vec = false;
    if (T_dst[e + 1] != T_dst[e] + 1 || (T_dst[e] & 1)) vec = false;
  }
  for (int i = 0; vec && i < pp.outer.n; ++i)
    if ((pp.outer.st0[i] & 1) || (pp.outer.st1[i] & 1)) vec = false;
  pp.vec = vec ? 1 : 0;
  return true;
}

int run_launches(Plan& P, const std::vector<Launch>& ls, cudaStream_t st, int stop_vertex) {
  for (const Launch& L : ls) {
    cudaError_t e = cudaSuccess;
    switch (L.type) {
      case L_GATHER:
        e = launch_gather(P.d_jobs, P.d_gstart, P.njobs, P.gather_blocks, P.pool, P.counter, st);
        break;
      case L_SIMT:
        e = launch_simt(P.simt[L.idx], st);
        break;
      case L_PACK:
        e = launch_pack(P.packs[L.idx], st);
        break;
      case L_PERM:
        e = launch_perm(P.perms[L.idx], st);
        break;
      case L_DOT: {
        const DotParams& dp = P.dots[L.idx];
        e = dp.perm >= 0 ? launch_perm_dot(P.perms[dp.perm], P.partial, dp.z, st) : launch_dot(dp, st);
        break;
      }
      case L_RENORM: {
        const TensorLoc& t = P.T[L.idx];
        unsigned int* bits = P.d_absmax + L.idx;
        e = launch_absmax(P.ptr(t), t.size, bits, st);
        if (e == cudaSuccess)
          e = launch_rescale(P.ptr(t), t.size, bits, P.d_exps + (P.V[L.idx - P.n].hoisted ? 0 : 1), st);
        break;
      }
      case L_RESET: {
        const int nv = P.n > 1 ? 2 * P.n - 1 : 1;
        e = cudaMemsetAsync(P.d_absmax, 0, nv * sizeof(unsigned int), st);
        if (e == cudaSuccess) e = cudaMemsetAsync(P.d_exps + L.idx, 0, sizeof(long long), st);
        break;
      }
      case L_SIMTB: {
        const Plan::SimtBatch& bt = P.batches[L.idx];
        e = launch_simt_batch(P.d_bjobs + bt.job_off, P.d_bstarts + bt.start_off, bt.njobs,
                              bt.total_blocks, st);
        if (e == cudaSuccess && stop_vertex >= 0 &&
            std::find(bt.vertices.begin(), bt.vertices.end(), stop_vertex) != bt.vertices.end())
          return TNX_OK;
        break;
      }
      case L_GEMM:
        e = launch_gemm(P.gemms[L.idx], st);
        break;
      case L_ACCUM:
        if (stop_vertex >= 0) continue;
        e = launch_accum(P.accum, st);
        break;
    }
    if (e != cudaSuccess) return fail(TNX_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
    if (stop_vertex >= 0 && L.vertex == stop_vertex && L.type != L_PACK && L.type != L_PERM &&
        L.type != L_RENORM)
      break;
  }
  return TNX_OK;
}

// Resolve pointers / tensor maps of every launch.  Requires arenas.
int lower(Plan& P) {
  std::string err;
  char ebuf[256];
  P.simt.clear();
  P.packs.clear();
  P.perms.clear();
  P.dots.clear();
  P.ptabs.clear();
  P.gemms.clear();
  P.hoist_launches.clear();
  P.slice_launches.clear();
  if (!P.gather_leaves.empty()) P.slice_launches.push_back({L_GATHER, 0, -1});
  P.batches.clear();
  P.bjobs.clear();
  P.bstarts.clear();
  for (int phase = 0; phase < 2; ++phase) {
    const std::vector<int>& order = phase == 0 ? P.hoist_order : P.slice_order;
    std::vector<Launch>& out = phase == 0 ? P.hoist_launches : P.slice_launches;
    if (P.strip()) out.push_back({L_RESET, phase, -1});
    int open_batch = -1, batch_level = -1;
    std::vector<int> pending_renorm;  // strip_exponent: batched vertices of the open level
    size_t renorm_mark = 0;
    for (int k : order) {
      Vertex& v = P.V[k];
      if (P.level[k] != batch_level) {
        for (int pv : pending_renorm) out.push_back({L_RENORM, pv, pv});
        pending_renorm.clear();
        open_batch = -1;
        batch_level = P.level[k];
      }
      renorm_mark = out.size();
      const TensorLoc& x = P.T[v.a];
      const TensorLoc& y = P.T[v.b];
      const TensorLoc& z = P.T[v.ssa];
      if (v.kind == VK_GEMM) {
        float* apl = reinterpret_cast<float*>(P.block_ptr(phase, v.blk_apl));
        float* bpl = reinterpret_cast<float*>(P.block_ptr(phase, v.blk_bpl));
        std::vector<int> rows_a = v.bl;
        rows_a.insert(rows_a.end(), v.ml.begin(), v.ml.end());
        std::vector<int> rows_b = v.bl;
        rows_b.insert(rows_b.end(), v.nl.begin(), v.nl.end());
        if (v.swap) std::swap(rows_a, rows_b);
        const TensorLoc& opa = v.swap ? y : x;
        const TensorLoc& opb = v.swap ? x : y;
        const int64_t ra = v.swap ? v.N : v.M, rb = v.swap ? v.M : v.N;
        for (int side = 0; side < 2; ++side) {
          const TensorLoc& src = side == 0 ? opa : opb;
          const std::vector<int>& rows = side == 0 ? rows_a : rows_b;
          float* planes = side == 0 ? apl : bpl;
          const int64_t nrows = v.B * (side == 0 ? ra : rb);
          bool done = false;
          if (v.side_direct[side]) continue;  // written by the child GEMM's epilogue
          std::vector<int> dst;
          if (plane_order(P, v, side, dst) && !(P.flags & TNX_FLAG_NO_TILED_PACK)) {
            PermParams pp;
            int64_t toff = 0;
            const size_t mark = P.ptabs.size();
            const bool mixp = P.precision == TNX_PREC_TF32_BF16X;
            const int pmode = mixp ? (side == 0 ? 3 : 4) : (side == 1 && v.stack ? 2 : 1);
            if (build_perm(P, src, dst, pmode, pp, toff, err)) {
              pp.src = P.ptr(src);
              pp.dst = planes;
              pp.plane_stride = nrows * v.kp;
              if ((pp.plane_stride & 1) || (src.arena == AR_POOL && (src.offset & 1))) pp.vec = 0;
              pp.tab = reinterpret_cast<const int32_t*>(toff);  // rebased after upload
              P.perms.push_back(pp);
              out.push_back({L_PERM, (int)P.perms.size() - 1, v.ssa});
              done = true;
            } else {
              P.ptabs.resize(mark);
            }
          }
          if (!done) {
            PackParams pk{};
            if (!build_map(P, rows, &src, nullptr, pk.row, err) || !build_map(P, v.cl, &src, nullptr, pk.col, err))
              return fail(TNX_ERR_INVALID, "vertex " + std::to_string(v.ssa) + ": " + err);
            pk.src = P.ptr(src);
            pk.dst = planes;
            pk.rows = nrows;
            pk.K = v.K;
            pk.kp = v.kp;
            pk.plane_stride = nrows * v.kp;
            pk.nplanes = side == 1 && v.stack ? 6 : 4;
            pk.mix = P.precision == TNX_PREC_TF32_BF16X ? (side == 0 ? 1 : 2) : 0;
            P.packs.push_back(pk);
            out.push_back({L_PACK, (int)P.packs.size() - 1, v.ssa});
          }
        }
        GemmPlan g;
        float2* part = v.splits > 1 ? reinterpret_cast<float2*>(P.block_ptr(phase, v.blk_part)) : nullptr;
        if (gemm_prepare(&g, apl, bpl, P.ptr(z), v.B, ra, rb, v.kp, v.splits, part, ebuf, sizeof(ebuf),
                         v.stack ? 1 : 0))
          return fail(TNX_ERR_CUDA, std::string("vertex ") + std::to_string(v.ssa) + ": " + ebuf);
        if (g.two_sm != v.two_sm)
          return fail(TNX_ERR_INVALID, "vertex " + std::to_string(v.ssa) + ": GEMM configuration changed");
        g.mix = P.precision == TNX_PREC_TF32_BF16X ? 1 : 0;
        if (v.direct_parent >= 0) {
          const Vertex& pv = P.V[v.direct_parent - P.n];
          std::vector<int> pdst;
          if (!plane_order(P, pv, v.direct_side, pdst))
            return fail(TNX_ERR_INVALID, "direct planes: parent layout changed");
          TensorLoc pl;
          pl.labels = pdst;  // row-major strides of the parent's plane order
          std::vector<int> crow = v.bl;
          const std::vector<int>& first = v.swap ? v.nl : v.ml;
          const std::vector<int>& second = v.swap ? v.ml : v.nl;
          crow.insert(crow.end(), first.begin(), first.end());
          if (!build_map(P, crow, &pl, nullptr, g.fmap, err) || !build_map(P, second, &pl, nullptr, g.gmap, err))
            return fail(TNX_ERR_INVALID, "vertex " + std::to_string(v.ssa) + ": " + err);
          const int64_t prows = pv.B * (v.direct_side == 0 ? (pv.swap ? pv.N : pv.M) : (pv.swap ? pv.M : pv.N));
          g.direct = 1;
          g.dmix = g.mix;
          g.dside = v.direct_side;
          g.dstack = v.direct_side == 1 && pv.stack ? 1 : 0;
          g.dplanes = reinterpret_cast<float*>(
              P.block_ptr(phase, v.direct_side == 0 ? pv.blk_apl : pv.blk_bpl));
          g.dplane_stride = prows * pv.kp;
          // vector stores when every aligned group of 4 columns is contiguous
          {
            const IdxMap& gm = g.gmap;
            bool vec = gm.n >= 1 && gm.st0[gm.n - 1] == 1 && gm.dim[gm.n - 1] % 4 == 0 && (v.N % 4) == 0 &&
                       (g.dplane_stride % 4) == 0;
            for (int i = 0; vec && i < gm.n - 1; ++i)
              if (gm.st0[i] % 4) vec = false;
            for (int i = 0; vec && i < g.fmap.n; ++i)
              if (g.fmap.st0[i] % 4) vec = false;
            g.dvec = vec ? 1 : 0;
            // paired full-line stores (EPI 1): rows contiguous in groups of 16 and
            // column pairs 16 floats apart
            const IdxMap& fm = g.fmap;
            int64_t e = 1;
            bool rows16 = fm.n >= 1;
            for (int i = fm.n - 1; rows16 && i >= 0 && e < 16; --i) {
              if (fm.st0[i] != e) rows16 = false;
              e *= fm.dim[i];
            }
            const int64_t ra_rows = v.swap ? v.N : v.M;
            g.dpair = !vec && rows16 && e >= 16 && ra_rows % 32 == 0 && gm.n >= 1 && gm.st0[gm.n - 1] == 16 &&
                              gm.dim[gm.n - 1] % 2 == 0 && !g.mix && !dpair_off()
                          ? 1 : 0;
          }
        }
        P.gemms.push_back(g);
        out.push_back({L_GEMM, (int)P.gemms.size() - 1, v.ssa});
      } else if (v.kind == VK_DOT) {
        const float2* yp = P.ptr(y);
        if (v.blk_tmp >= 0) {
          PermParams pp;
          int64_t toff = 0;
          float2* tmp = reinterpret_cast<float2*>(P.block_ptr(phase, v.blk_tmp));
          if (!build_perm(P, y, x.labels, 0, pp, toff, err))
            return fail(TNX_ERR_INVALID, "vertex " + std::to_string(v.ssa) + ": dot permute: " + err);
          pp.src = yp;
          pp.dst = tmp;
          if ((y.arena == AR_POOL && (y.offset & 1)) || (x.arena == AR_POOL && (x.offset & 1))) pp.vec = 0;
          pp.tab = reinterpret_cast<const int32_t*>(toff);
          pp.dotx = P.ptr(x);
          P.perms.push_back(pp);
          yp = tmp;
        }
        DotParams dp{};
        dp.x = P.ptr(x);
        dp.y = yp;
        dp.z = P.ptr(z);
        dp.partial = P.partial;
        dp.n = x.size;
        dp.nblocks = 148 * 8;
        // y in another layout: one fused launch reads y through the permute tile
        // and multiplies with x in place (no permuted copy of y)
        dp.perm = v.blk_tmp >= 0 ? (int)P.perms.size() - 1 : -1;
        P.dots.push_back(dp);
        out.push_back({L_DOT, (int)P.dots.size() - 1, v.ssa});
      } else {
        SimtParams s{};
        std::vector<int> sum = v.cl;
        sum.insert(sum.end(), v.dxl.begin(), v.dxl.end());
        sum.insert(sum.end(), v.dyl.begin(), v.dyl.end());
        if (!build_map(P, z.labels, &x, &y, s.out, err) || !build_map(P, sum, &x, &y, s.sum, err))
          return fail(TNX_ERR_INVALID, "vertex " + std::to_string(v.ssa) + ": " + err);
        s.x = P.ptr(x);
        s.y = P.ptr(y);
        s.z = P.ptr(z);
        s.out_size = z.size;
        s.sum_size = v.sum_size;
        s.mode = v.kind;
        s.nsplit = v.nsplit;
        s.chunk = v.chunk;
        s.partial = P.partial;
        s.sum_tab = v.tab_off >= 0 ? P.d_tabs + v.tab_off : nullptr;
        s.group_lg = v.kind == VK_SIMT_W ? 5 : 0;
        if (v.plane_parent >= 0) {
          const Vertex& pv = P.V[v.plane_parent - P.n];
          std::vector<int> pdst;
          if (!plane_order(P, pv, v.plane_side, pdst))
            return fail(TNX_ERR_INVALID, "simt planes: parent layout changed");
          TensorLoc pl;
          pl.labels = pdst;
          if (!build_map(P, z.labels, &pl, nullptr, s.zmap, err))
            return fail(TNX_ERR_INVALID, "vertex " + std::to_string(v.ssa) + ": " + err);
          const int64_t pra = pv.swap ? pv.N : pv.M, prb = pv.swap ? pv.M : pv.N;
          s.zplanes = reinterpret_cast<float*>(P.block_ptr(phase, v.plane_side == 0 ? pv.blk_apl : pv.blk_bpl));
          s.zps = pv.B * (v.plane_side == 0 ? pra : prb) * pv.kp;
          s.znp = v.plane_side == 1 && pv.stack ? 6 : 4;
        }
        if (v.kind == VK_SIMT_T && s.sum.n == 1 && v.sum_size >= 2 &&
            (s.sum.st0[0] == 1 || s.sum.st1[0] == 1)) {
          // the summed run is contiguous in an operand: 2^lg lanes per output read it coalesced
          static const int gmax = getenv("TNX_SIMT_GROUP_LG") ? atoi(getenv("TNX_SIMT_GROUP_LG")) : 0;
          int lg = 0;
          while (lg < gmax && (int64_t(2) << lg) <= v.sum_size) ++lg;
          s.group_lg = lg;
        }
        if (v.kind == VK_SIMT_T || v.kind == VK_SIMT_W) {
          // one launch per dependency level for all its small contractions
          if (open_batch < 0) {
            P.batches.push_back(Plan::SimtBatch());
            open_batch = (int)P.batches.size() - 1;
            P.batches[open_batch].job_off = (int64_t)P.bjobs.size();
            out.push_back({L_SIMTB, open_batch, -1});
          }
          Plan::SimtBatch& bt = P.batches[open_batch];
          bt.vertices.push_back(v.ssa);
          bt.njobs++;
          P.bjobs.push_back(s);
          if (P.strip()) pending_renorm.push_back(v.ssa);
          continue;
        }
        P.simt.push_back(s);
        out.push_back({L_SIMT, (int)P.simt.size() - 1, v.ssa});
      }
      if (P.strip() && out.size() > renorm_mark) out.push_back({L_RENORM, v.ssa, v.ssa});
    }
    for (int pv : pending_renorm) out.push_back({L_RENORM, pv, pv});
  }
  // accumulate: root -> output order
  const int root = P.n > 1 ? 2 * P.n - 2 : 0;
  const TensorLoc& r = P.T[root];
  std::vector<int> extra;
  for (int l : r.labels)
    if (std::find(P.output.begin(), P.output.end(), l) == P.output.end()) extra.push_back(l);
  std::memset(&P.accum, 0, sizeof(P.accum));
  if (!build_map(P, P.output, &r, nullptr, P.accum.out, err) || !build_map(P, extra, &r, nullptr, P.accum.extra, err))
    return fail(TNX_ERR_INVALID, "accumulate: " + err);
  P.accum.root = P.ptr(r);
  P.accum.acc = P.acc;
  P.accum.comp = P.comp;
  P.accum.out_size = P.out_size;
  P.accum.extra_size = P.prod(extra);
  P.accum.slice_counter = P.counter;
  if (P.strip()) {
    P.accum.hoist_exp = P.d_exps;
    P.accum.slice_exp = P.d_exps + 1;
    P.accum.acc_exp = P.d_acc_exp;
  }
  P.slice_launches.push_back({L_ACCUM, 0, -1});
  return TNX_OK;
}

// Precomputed summed-index offset tables (int32) for small SIMT sums.
void build_tables(Plan& P) {
  P.tables.clear();
  for (auto& v : P.V) {
    v.tab_off = -1;
    if (v.kind == VK_GEMM || v.kind == VK_SIMT_S || v.kind == VK_DOT || v.sum_size > 4096) continue;
    const TensorLoc& x = P.T[v.a];
    const TensorLoc& y = P.T[v.b];
    std::vector<int> sum = v.cl;
    sum.insert(sum.end(), v.dxl.begin(), v.dxl.end());
    sum.insert(sum.end(), v.dyl.begin(), v.dyl.end());
    std::vector<int64_t> sx, sy, dm;
    for (int l : sum) {
      dm.push_back(P.dims[l]);
      sx.push_back(P.stride_in(x, l));
      sy.push_back(P.stride_in(y, l));
    }
    bool fits = x.size < (int64_t(1) << 31) && y.size < (int64_t(1) << 31);
    if (!fits) continue;
    v.tab_off = (int64_t)P.tables.size();
    std::vector<int64_t> dig(dm.size(), 0);
    for (int64_t j = 0; j < v.sum_size; ++j) {
      int64_t ox = 0, oy = 0;
      for (size_t i = 0; i < dm.size(); ++i) {
        ox += dig[i] * sx[i];
        oy += dig[i] * sy[i];
      }
      P.tables.push_back({(int32_t)ox, (int32_t)oy});
      for (int i = (int)dm.size() - 1; i >= 0; --i) {
        if (++dig[i] < dm[i]) break;
        dig[i] = 0;
      }
    }
  }
}

}  // namespace

// Order stream `st` after the plan's previous work (if it ran on another stream).
static int order_after(Plan& P, cudaStream_t st) {
  if (P.order_valid && P.last_stream != st) TNX_CUDA(cudaStreamWaitEvent(st, P.order_ev, 0));
  return TNX_OK;
}

// Record the end of this call's work on `st` for the next call to order after.
static int mark_done(Plan& P, cudaStream_t st) {
  if (!P.order_ev) TNX_CUDA(cudaEventCreateWithFlags(&P.order_ev, cudaEventDisableTiming));
  TNX_CUDA(cudaEventRecord(P.order_ev, st));
  P.last_stream = st;
  P.order_valid = true;
  return TNX_OK;
}

extern "C" {

const char* tnx_last_error(void) { return g_err.c_str(); }
const char* tnx_version(void) { return "tnx 0.1 (sm_100a, tcgen05 split-TF32)"; }

int tnx_plan_create(const tnx_plan_desc* desc, void** plan_out) {
  if (!desc || !plan_out) return fail(TNX_ERR_INVALID, "null argument");
  std::unique_ptr<Plan> P(new Plan());
  int rc = compile(*P, desc);
  if (rc) return rc;
  if (!P->too_wide) build_tables(*P);
  *plan_out = P.release();
  return TNX_OK;
}

int tnx_plan_destroy(void* plan) {
  if (!plan) return TNX_OK;
  Plan* P = static_cast<Plan*>(plan);
  if (P->bound) cudaSetDevice(P->device);
  delete P;
  return TNX_OK;
}

int tnx_bind_leaves(void* plan, const void* const* leaf_data, int32_t dtype, int32_t location,
                    void* stream) {
  if (!plan || !leaf_data) return fail(TNX_ERR_INVALID, "null argument");
  Plan& P = *static_cast<Plan*>(plan);
  if (P.too_wide)
    return fail(TNX_ERR_OOM, "W_s=" + std::to_string(P.width) + " cannot be executed; slice more labels");
  TNX_CUDA(cudaSetDevice(P.device));
  if (!P.bound) {
    char ebuf[256];
    if (P.precision != TNX_PREC_FP32 && gemm_init_attributes(ebuf, sizeof(ebuf)))
      return fail(TNX_ERR_CUDA, ebuf);
    size_t free_b = 0, total_b = 0;
    TNX_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const int64_t need = P.pool_elems * 8 + P.work_bytes + P.persist_bytes + P.max_partial * 8 +
                         (int64_t)P.tables.size() * 8 + P.out_size * 32;
    if ((double)need > 0.97 * (double)free_b)
      return fail(TNX_ERR_OOM, "plan needs " + std::to_string(need) + " bytes of HBM, " +
                                   std::to_string(free_b) + " free");
    TNX_CUDA(cudaStreamCreateWithFlags(&P.own, cudaStreamNonBlocking));
    TNX_CUDA(cudaMalloc(&P.pool, P.pool_elems * 8));
    TNX_CUDA(cudaMalloc(&P.work, P.work_bytes));
    TNX_CUDA(cudaMalloc(&P.persist, P.persist_bytes));
    if (P.max_partial) TNX_CUDA(cudaMalloc(&P.partial, P.max_partial * 8));
    if (!P.tables.empty()) {
      TNX_CUDA(cudaMalloc(&P.d_tabs, P.tables.size() * sizeof(Int2Off)));
      TNX_CUDA(cudaMemcpy(P.d_tabs, P.tables.data(), P.tables.size() * sizeof(Int2Off), cudaMemcpyHostToDevice));
    }
    TNX_CUDA(cudaMalloc(&P.acc, std::max<int64_t>(P.out_size, 1) * 16));
    TNX_CUDA(cudaMalloc(&P.comp, std::max<int64_t>(P.out_size, 1) * 16));
    TNX_CUDA(cudaMalloc(&P.counter, 8));
    if (P.strip()) {
      const int nvv = P.n > 1 ? 2 * P.n - 1 : 1;
      TNX_CUDA(cudaMalloc(&P.d_absmax, nvv * sizeof(unsigned int)));
      TNX_CUDA(cudaMalloc(&P.d_exps, 2 * sizeof(long long)));
      TNX_CUDA(cudaMemset(P.d_exps, 0, 2 * sizeof(long long)));
      TNX_CUDA(cudaMalloc(&P.d_acc_exp, std::max<int64_t>(P.out_size, 1) * sizeof(long long)));
    }
    // gather jobs
    std::vector<GatherJob> jobs;
    for (int i : P.gather_leaves) {
      GatherJob j{};
      const std::vector<int>& ls = P.leaf_labels[i];
      j.src = P.pool_off[i];
      j.dst = reinterpret_cast<float2*>(P.block_ptr(1, P.T[i].block));
      j.out_size = P.T[i].size;
      int64_t s = 1;
      std::vector<int64_t> st(ls.size());
      for (int q = (int)ls.size() - 1; q >= 0; --q) {
        st[q] = s;
        s *= P.dims[ls[q]];
      }
      for (size_t q = 0; q < ls.size(); ++q) {
        int l = ls[q];
        const bool merge = P.slice_pos[l] < 0 && j.n_kept > 0 && j.kst[j.n_kept - 1] == st[q] * P.dims[l];
        if (!merge && (P.slice_pos[l] >= 0 ? j.n_sl : j.n_kept) >= kMaxLeafRank)
          return fail(TNX_ERR_INVALID, "leaf " + std::to_string(i) + ": more than " + std::to_string(kMaxLeafRank) +
                                           " sliced labels or non-contiguous kept runs");
        if (P.slice_pos[l] >= 0) {
          u128 rad = 1;
          for (size_t t = P.slice_pos[l] + 1; t < P.sliced.size(); ++t) rad *= (u128)P.dims[P.sliced[t]];
          j.radix[j.n_sl] = (uint64_t)rad;
          j.sdim[j.n_sl] = P.dims[l];
          j.sst[j.n_sl] = st[q];
          j.n_sl++;
        } else if (merge) {
          j.kdim[j.n_kept - 1] *= P.dims[l];  // merge into the previous contiguous run
          j.kst[j.n_kept - 1] = st[q];
        } else {
          j.kdim[j.n_kept] = P.dims[l];
          j.kst[j.n_kept] = st[q];
          j.n_kept++;
        }
      }
      {
        bool v = j.n_kept > 0 && j.kst[j.n_kept - 1] == 1 && j.kdim[j.n_kept - 1] % 2 == 0 && j.src % 2 == 0 &&
                 reinterpret_cast<uintptr_t>(j.dst) % 16 == 0;
        for (int q = 0; v && q < j.n_kept - 1; ++q) v = j.kst[q] % 2 == 0;
        for (int q = 0; v && q < j.n_sl; ++q) v = j.sst[q] % 2 == 0;
        j.vec = v ? 1 : 0;
      }
      jobs.push_back(j);
    }
    P.njobs = (int)jobs.size();
    if (P.njobs) {
      std::vector<int32_t> gstart(1, 0);
      for (const GatherJob& j : jobs) {
        const int64_t nb = std::min<int64_t>(148 * 8, std::max<int64_t>(1, (j.out_size + 1023) / 1024));
        gstart.push_back(gstart.back() + (int32_t)nb);
      }
      P.gather_blocks = gstart.back();
      TNX_CUDA(cudaMalloc(&P.d_jobs, jobs.size() * sizeof(GatherJob)));
      TNX_CUDA(cudaMemcpy(P.d_jobs, jobs.data(), jobs.size() * sizeof(GatherJob), cudaMemcpyHostToDevice));
      TNX_CUDA(cudaMalloc(&P.d_gstart, gstart.size() * sizeof(int32_t)));
      TNX_CUDA(cudaMemcpy(P.d_gstart, gstart.data(), gstart.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    int rc = lower(P);
    if (rc) return rc;
    for (auto& bt : P.batches) {
      bt.start_off = (int64_t)P.bstarts.size();
      int acc_blocks = 0;
      for (int j = 0; j < bt.njobs; ++j) {
        P.bstarts.push_back(acc_blocks);
        acc_blocks += simt_blocks(P.bjobs[bt.job_off + j]);
      }
      P.bstarts.push_back(acc_blocks);
      bt.total_blocks = acc_blocks;
    }
    if (!P.bjobs.empty()) {
      TNX_CUDA(cudaMalloc(&P.d_bjobs, P.bjobs.size() * sizeof(SimtParams)));
      TNX_CUDA(cudaMemcpy(P.d_bjobs, P.bjobs.data(), P.bjobs.size() * sizeof(SimtParams), cudaMemcpyHostToDevice));
      TNX_CUDA(cudaMalloc(&P.d_bstarts, P.bstarts.size() * sizeof(int32_t)));
      TNX_CUDA(cudaMemcpy(P.d_bstarts, P.bstarts.data(), P.bstarts.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    }
    if (!P.ptabs.empty()) {
      TNX_CUDA(cudaMalloc(&P.d_ptabs, P.ptabs.size() * sizeof(int32_t)));
      TNX_CUDA(cudaMemcpy(P.d_ptabs, P.ptabs.data(), P.ptabs.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      for (auto& pp : P.perms) pp.tab = P.d_ptabs + reinterpret_cast<intptr_t>(pp.tab);
    }
    P.bound = true;
  }
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.own;
  if (int orc = order_after(P, st)) return orc;
  // upload leaves
  int64_t max_leaf = 0;
  for (int i = 0; i < P.n; ++i) max_leaf = std::max<int64_t>(max_leaf, P.prod(P.leaf_labels[i]));
  if (location == TNX_LOC_HOST) {
    if (dtype == TNX_DTYPE_C128) {
      if (!P.staging) {
        TNX_CUDA(cudaMallocHost(&P.staging, P.pool_elems * 8));
        std::memset(P.staging, 0, P.pool_elems * 8);
      }
      // the previous upload (on whichever stream) finished reading the staging buffer
      TNX_CUDA(cudaStreamSynchronize(st));
      if (P.order_valid) TNX_CUDA(cudaEventSynchronize(P.order_ev));
      for (int i = 0; i < P.n; ++i) {
        const double* src = static_cast<const double*>(leaf_data[i]);
        int64_t sz = P.prod(P.leaf_labels[i]);
        for (int64_t e = 0; e < sz; ++e)
          P.staging[P.pool_off[i] + e] = make_float2((float)src[2 * e], (float)src[2 * e + 1]);
      }
      TNX_CUDA(cudaMemcpyAsync(P.pool, P.staging, P.pool_elems * 8, cudaMemcpyHostToDevice, st));
    } else {
      for (int i = 0; i < P.n; ++i)
        TNX_CUDA(cudaMemcpyAsync(P.pool + P.pool_off[i], leaf_data[i], P.prod(P.leaf_labels[i]) * 8,
                                 cudaMemcpyHostToDevice, st));
    }
  } else {
    for (int i = 0; i < P.n; ++i) {
      int64_t sz = P.prod(P.leaf_labels[i]);
      if (dtype == TNX_DTYPE_C128) {
        cudaError_t e = launch_convert_c128(static_cast<const double2*>(leaf_data[i]), P.pool + P.pool_off[i], sz, st);
        if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
      } else {
        TNX_CUDA(cudaMemcpyAsync(P.pool + P.pool_off[i], leaf_data[i], sz * 8, cudaMemcpyDeviceToDevice, st));
      }
    }
  }
  (void)max_leaf;
  // hoisted (slice-invariant) subtrees, computed once per bind; captured as a
  // graph on the first bind (fixed buffers) and replayed by later re-binds
  int rc = 0;
  if (!(P.flags & TNX_FLAG_NO_GRAPH) && !P.hoist_launches.empty()) {
    if (!P.hgexec) {
      cudaStream_t cs = P.own;
      TNX_CUDA(cudaStreamSynchronize(st));
      TNX_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      rc = run_launches(P, P.hoist_launches, cs, -1);
      cudaGraph_t g = nullptr;
      cudaError_t ce = cudaStreamEndCapture(cs, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (ce != cudaSuccess) return fail(TNX_ERR_CUDA, std::string("hoist graph capture: ") + cudaGetErrorString(ce));
      P.hgraph = g;
      TNX_CUDA(cudaGraphInstantiate(&P.hgexec, g, 0));
    }
    TNX_CUDA(cudaGraphLaunch(P.hgexec, st));
  } else {
    rc = run_launches(P, P.hoist_launches, st, -1);
    if (rc) return rc;
  }
  TNX_CUDA(cudaMemsetAsync(P.acc, 0, std::max<int64_t>(P.out_size, 1) * 16, st));
  TNX_CUDA(cudaMemsetAsync(P.comp, 0, std::max<int64_t>(P.out_size, 1) * 16, st));
  if (P.d_acc_exp) TNX_CUDA(cudaMemsetAsync(P.d_acc_exp, 0, std::max<int64_t>(P.out_size, 1) * 8, st));
  // per-slice graph
  if (!(P.flags & TNX_FLAG_NO_GRAPH) && !P.gexec) {
    cudaStream_t cs = P.own;
    TNX_CUDA(cudaStreamSynchronize(st));
    TNX_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    rc = run_launches(P, P.slice_launches, cs, -1);
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(cs, &g);
    if (rc) return rc;
    if (ce != cudaSuccess) return fail(TNX_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
    P.graph = g;
    TNX_CUDA(cudaGraphInstantiate(&P.gexec, g, 0));
  }
  return mark_done(P, st);
}

int tnx_run_slices(void* plan, uint64_t s_begin, uint64_t s_end, void* stream) {
  if (!plan) return fail(TNX_ERR_INVALID, "null plan");
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "tnx_run_slices before tnx_bind_leaves");
  if ((u128)s_end > P.d || s_begin > s_end) return fail(TNX_ERR_INVALID, "slice range out of [0, d)");
  TNX_CUDA(cudaSetDevice(P.device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.own;
  if (s_begin == s_end) return TNX_OK;
  if (int orc = order_after(P, st)) return orc;
  cudaError_t e = launch_set_counter(P.counter, s_begin, st);
  if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
  for (uint64_t s = s_begin; s < s_end; ++s) {
    if (P.gexec) {
      TNX_CUDA(cudaGraphLaunch(P.gexec, st));
    } else {
      int rc = run_launches(P, P.slice_launches, st, -1);
      if (rc) return rc;
    }
  }
  return mark_done(P, st);
}

int tnx_run_slice_ids(void* plan, const uint64_t* ids, int64_t n, void* stream) {
  if (!plan) return fail(TNX_ERR_INVALID, "null plan");
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "tnx_run_slice_ids before tnx_bind_leaves");
  if (n < 0 || (n > 0 && !ids)) return fail(TNX_ERR_INVALID, "tnx_run_slice_ids: bad id list");
  for (int64_t i = 0; i < n; ++i)
    if ((u128)ids[i] >= P.d) return fail(TNX_ERR_INVALID, "slice id " + std::to_string(ids[i]) + " out of [0, d)");
  TNX_CUDA(cudaSetDevice(P.device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.own;
  if (n == 0) return TNX_OK;
  if (int orc = order_after(P, st)) return orc;
  // maximal runs of consecutive ids: one counter write, then graph replays
  // (the last kernel of each replay advances the device-side slice id)
  for (int64_t i = 0; i < n;) {
    int64_t j = i + 1;
    while (j < n && ids[j] == ids[j - 1] + 1) ++j;
    cudaError_t e = launch_set_counter(P.counter, ids[i], st);
    if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
    for (int64_t k = i; k < j; ++k) {
      if (P.gexec) {
        TNX_CUDA(cudaGraphLaunch(P.gexec, st));
      } else {
        int rc = run_launches(P, P.slice_launches, st, -1);
        if (rc) return rc;
      }
    }
    i = j;
  }
  return mark_done(P, st);
}

int tnx_reset_accumulator(void* plan, void* stream) {
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "not bound");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.own;
  if (int orc = order_after(P, st)) return orc;
  TNX_CUDA(cudaMemsetAsync(P.acc, 0, std::max<int64_t>(P.out_size, 1) * 16, st));
  TNX_CUDA(cudaMemsetAsync(P.comp, 0, std::max<int64_t>(P.out_size, 1) * 16, st));
  if (P.d_acc_exp) TNX_CUDA(cudaMemsetAsync(P.d_acc_exp, 0, std::max<int64_t>(P.out_size, 1) * 8, st));
  return mark_done(P, st);
}

int tnx_partial_result(void* plan, double* out, int64_t out_elems, void* stream) {
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "not bound");
  if (out_elems != P.out_size) return fail(TNX_ERR_INVALID, "output size mismatch");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.own;
  if (int orc = order_after(P, st)) return orc;
  TNX_CUDA(cudaMemcpyAsync(out, P.acc, P.out_size * 16, cudaMemcpyDeviceToHost, st));
  TNX_CUDA(cudaStreamSynchronize(st));
  return TNX_OK;
}

int tnx_partial_result_async(void* plan, double* out, int64_t out_elems, void* stream) {
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "not bound");
  if (out_elems != P.out_size) return fail(TNX_ERR_INVALID, "output size mismatch");
  if (!out) return fail(TNX_ERR_INVALID, "null output buffer");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.own;
  if (int orc = order_after(P, st)) return orc;
  TNX_CUDA(cudaMemcpyAsync(out, P.acc, P.out_size * 16, cudaMemcpyDeviceToHost, st));
  return mark_done(P, st);
}

int tnx_partial_result_exp(void* plan, double* out, int64_t* exp2, int64_t out_elems, void* stream) {
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "not bound");
  if (!P.strip()) return fail(TNX_ERR_STATE, "plan was not created with TNX_FLAG_STRIP_EXPONENT");
  if (out_elems != P.out_size) return fail(TNX_ERR_INVALID, "output size mismatch");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : P.own;
  if (int orc = order_after(P, st)) return orc;
  TNX_CUDA(cudaMemcpyAsync(out, P.acc, P.out_size * 16, cudaMemcpyDeviceToHost, st));
  TNX_CUDA(cudaMemcpyAsync(exp2, P.d_acc_exp, P.out_size * 8, cudaMemcpyDeviceToHost, st));
  TNX_CUDA(cudaStreamSynchronize(st));
  return TNX_OK;
}

int tnx_allreduce(void* const* plans, int32_t nplans, void* const* streams) {
  if (!plans || nplans < 1) return fail(TNX_ERR_INVALID, "tnx_allreduce: no plans");
  for (int i = 0; i < nplans; ++i) {
    if (!plans[i]) return fail(TNX_ERR_INVALID, "tnx_allreduce: null plan");
    for (int j = 0; j < i; ++j)
      if (plans[j] == plans[i]) return fail(TNX_ERR_INVALID, "tnx_allreduce: plan listed twice");
  }
  Plan& R = *static_cast<Plan*>(plans[0]);
  for (int i = 0; i < nplans; ++i) {
    const Plan& P = *static_cast<const Plan*>(plans[i]);
    if (!P.bound) return fail(TNX_ERR_STATE, "tnx_allreduce: plan " + std::to_string(i) + " not bound");
    if (P.out_size != R.out_size || P.strip() != R.strip())
      return fail(TNX_ERR_INVALID, "tnx_allreduce: plans differ in output size or strip_exponent mode");
  }
  auto stream_of = [&](int i) {
    Plan& P = *static_cast<Plan*>(plans[i]);
    return streams && streams[i] ? static_cast<cudaStream_t>(streams[i]) : P.own;
  };
  int prev = 0;
  TNX_CUDA(cudaGetDevice(&prev));
  const int n = nplans;
  const int64_t out = R.out_size;
  const bool strip = R.strip();
  const int64_t vbytes = out * 16, ebytes = out * 8;
  const int64_t need = (int64_t)n * (strip ? vbytes + ebytes : 2 * vbytes);
  cudaStream_t s0 = stream_of(0);
  TNX_CUDA(cudaSetDevice(R.device));
  if (R.ar_bytes < need) {
    if (R.ar_buf) TNX_CUDA(cudaFree(R.ar_buf));
    R.ar_buf = nullptr;
    TNX_CUDA(cudaMalloc(&R.ar_buf, need));
    R.ar_bytes = need;
  }
  char* buf = static_cast<char*>(R.ar_buf);
  double2* g_acc = reinterpret_cast<double2*>(buf);
  double2* g_comp = strip ? nullptr : reinterpret_cast<double2*>(buf + n * vbytes);
  long long* g_exp = strip ? reinterpret_cast<long long*>(buf + n * vbytes) : nullptr;
  std::vector<cudaEvent_t> evs(n, nullptr);
  auto cleanup = [&]() {
    for (int i = 0; i < n; ++i)
      if (evs[i]) {
        cudaSetDevice(static_cast<Plan*>(plans[i])->device);
        cudaEventDestroy(evs[i]);
      }
    cudaSetDevice(prev);
  };
  auto copy = [&](void* dst, int ddev, const void* src, int sdev, int64_t bytes) {
    return ddev == sdev ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s0)
                        : cudaMemcpyPeerAsync(dst, ddev, src, sdev, bytes, s0);
  };
  cudaError_t e = cudaSuccess;
  // 1. order after every plan's pending work, gather its partial into the root buffer
  for (int i = 0; i < n && e == cudaSuccess; ++i) {
    Plan& P = *static_cast<Plan*>(plans[i]);
    e = cudaSetDevice(P.device);
    if (e == cudaSuccess && P.order_valid && P.last_stream != stream_of(i))
      e = cudaStreamWaitEvent(stream_of(i), P.order_ev, 0);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(evs[i], stream_of(i));
    if (e == cudaSuccess) e = cudaSetDevice(R.device);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, evs[i], 0);
    if (e == cudaSuccess) e = copy(g_acc + i * out, R.device, P.acc, P.device, vbytes);
    if (e == cudaSuccess && strip) e = copy(g_exp + i * out, R.device, P.d_acc_exp, P.device, ebytes);
    if (e == cudaSuccess && !strip) e = copy(g_comp + i * out, R.device, P.comp, P.device, vbytes);
  }
  // 2. reduce on the root device into the root's accumulator
  if (e == cudaSuccess) e = cudaSetDevice(R.device);
  if (e == cudaSuccess)
    e = launch_allreduce(g_acc, g_comp, g_exp, n, out, R.acc, strip ? nullptr : R.comp,
                         strip ? R.d_acc_exp : nullptr, s0);
  // 3. broadcast the total back; every plan's stream waits for the exchange
  for (int i = 1; i < n && e == cudaSuccess; ++i) {
    Plan& P = *static_cast<Plan*>(plans[i]);
    e = copy(P.acc, P.device, R.acc, R.device, vbytes);
    if (e == cudaSuccess && strip) e = copy(P.d_acc_exp, P.device, R.d_acc_exp, R.device, ebytes);
    if (e == cudaSuccess && !strip) e = copy(P.comp, P.device, R.comp, R.device, vbytes);
  }
  if (e == cudaSuccess) e = cudaEventRecord(evs[0], s0);
  for (int i = 1; i < n && e == cudaSuccess; ++i) {
    e = cudaSetDevice(static_cast<Plan*>(plans[i])->device);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream_of(i), evs[0], 0);
  }
  // later calls on other streams order after the exchange
  for (int i = 0; i < n && e == cudaSuccess; ++i) {
    Plan& P = *static_cast<Plan*>(plans[i]);
    e = cudaSetDevice(P.device);
    if (e == cudaSuccess && !P.order_ev) e = cudaEventCreateWithFlags(&P.order_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(P.order_ev, stream_of(i));
    if (e == cudaSuccess) {
      P.last_stream = stream_of(i);
      P.order_valid = true;
    }
  }
  // events may be destroyed once recorded/waited on (resources are released on completion)
  cleanup();
  if (e != cudaSuccess) return fail(TNX_ERR_CUDA, std::string("tnx_allreduce: ") + cudaGetErrorString(e));
  return TNX_OK;
}

int tnx_stats_get(void* plan, tnx_stats* s) {
  if (!plan || !s) return fail(TNX_ERR_INVALID, "null argument");
  Plan& P = *static_cast<Plan*>(plan);
  std::memset(s, 0, sizeof(*s));
  s->op_count_lo = (uint64_t)P.ops;
  s->op_count_hi = (uint64_t)(P.ops >> 64);
  s->d_lo = (uint64_t)P.d;
  s->d_hi = (uint64_t)(P.d >> 64);
  s->width = P.width;
  s->peak_elements = P.peak > (u128)~0ull ? ~0ull : (uint64_t)P.peak;
  s->work_arena_bytes = P.work_bytes;
  s->persistent_bytes = P.persist_bytes;
  s->leaf_bytes = P.pool_elems * 8;
  s->num_vertices = P.n - 1;
  s->num_hoisted = (int)P.hoist_order.size();
  int ng = 0, ns = 0, launches = P.gather_leaves.empty() ? 1 : 2;
  for (int k : P.slice_order) {
    if (P.V[k].kind == VK_GEMM) {
      ++ng;
      launches += (P.V[k].splits > 1 ? 4 : 3) - (int)P.V[k].side_direct[0] - (int)P.V[k].side_direct[1];
    } else {
      ++ns;
      launches += P.V[k].kind == VK_SIMT_S ? 2 : P.V[k].kind == VK_DOT ? (P.V[k].blk_tmp >= 0 ? 3 : 2) : 1;
    }
  }
  s->num_gemm = ng;
  s->num_simt = ns;
  if (P.bound) {
    launches = 0;
    for (const Launch& L : P.slice_launches)
      launches += (L.type == L_GEMM && P.gemms[L.idx].splits > 1) || L.type == L_DOT ||
                          (L.type == L_SIMT && P.simt[L.idx].mode == SIMT_SPLIT)
                      ? 2
                      : 1;
  }
  s->launches_per_slice = launches;
  s->out_rank = (int)P.output.size();
  s->out_elements = P.out_size;
  return TNX_OK;
}

int tnx_vertex_info_get(void* plan, int32_t index, tnx_vertex_info* out) {
  Plan& P = *static_cast<Plan*>(plan);
  if (index < 0 || index >= (int)P.V.size()) return fail(TNX_ERR_INVALID, "vertex index out of range");
  const Vertex& v = P.V[index];
  out->ssa = v.ssa;
  out->kind = v.kind;
  out->hoisted = v.hoisted;
  out->rank = (int)P.T[v.ssa].labels.size();
  out->m = v.M;
  out->n = v.N;
  out->k = v.K;
  out->batch = v.B;
  out->macs_lo = (uint64_t)v.macs;
  out->macs_hi = (uint64_t)(v.macs >> 64);
  return TNX_OK;
}

int tnx_debug_vertex(void* plan, uint64_t s, int32_t v, float* out_c64, int64_t out_elems,
                     int32_t* layout_labels, int32_t* rank_out) {
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "not bound");
  const int nv = P.n > 1 ? 2 * P.n - 1 : 1;
  if (v < P.n || v >= nv) return fail(TNX_ERR_INVALID, "vertex must be internal");
  if ((u128)s >= P.d) return fail(TNX_ERR_INVALID, "slice out of range");
  const TensorLoc& t = P.T[v];
  if (t.fused)
    return fail(TNX_ERR_STATE, "vertex " + std::to_string(v) +
                                   " is fused into its parent's operand planes (plan with TNX_FLAG_NO_DIRECT to dump it)");
  if (out_elems != t.size) return fail(TNX_ERR_INVALID, "size mismatch: need " + std::to_string(t.size));
  TNX_CUDA(cudaSetDevice(P.device));
  cudaStream_t st = P.own;
  if (int orc = order_after(P, st)) return orc;
  TNX_CUDA(cudaStreamSynchronize(st));
  const Vertex& vx = P.V[v - P.n];
  int rc;
  if (vx.hoisted) {
    rc = run_launches(P, P.hoist_launches, st, v);
  } else {
    cudaError_t e = launch_set_counter(P.counter, s, st);
    if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
    rc = run_launches(P, P.slice_launches, st, v);
  }
  if (rc) return rc;
  TNX_CUDA(cudaMemcpyAsync(out_c64, P.ptr(t), t.size * 8, cudaMemcpyDeviceToHost, st));
  if (int mrc = mark_done(P, st)) return mrc;
  TNX_CUDA(cudaStreamSynchronize(st));
  for (size_t i = 0; i < t.labels.size(); ++i) layout_labels[i] = t.labels[i];
  *rank_out = (int)t.labels.size();
  return TNX_OK;
}

int tnx_profile_slice(void* plan, uint64_t s, int32_t* types, int32_t* vertices, float* ms,
                      double* alg_bytes, int32_t max_launches, int32_t* count) {
  Plan& P = *static_cast<Plan*>(plan);
  if (!P.bound) return fail(TNX_ERR_STATE, "not bound");
  if ((u128)s >= P.d) return fail(TNX_ERR_INVALID, "slice out of range");
  TNX_CUDA(cudaSetDevice(P.device));
  cudaStream_t st = P.own;
  if (int orc = order_after(P, st)) return orc;
  const int n = (int)P.slice_launches.size();
  std::vector<cudaEvent_t> ev(n + 1);
  for (auto& e : ev) TNX_CUDA(cudaEventCreate(&e));
  cudaError_t e = launch_set_counter(P.counter, s, st);
  if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
  TNX_CUDA(cudaEventRecord(ev[0], st));
  int done = 0;
  for (int i = 0; i < n; ++i) {
    const Launch& L = P.slice_launches[i];
    if (L.type == L_ACCUM) break;  // profiling does not accumulate
    std::vector<Launch> one{L};
    int rc = run_launches(P, one, st, -1);
    if (rc) return rc;
    TNX_CUDA(cudaEventRecord(ev[i + 1], st));
    done = i + 1;
  }
  if (int mrc = mark_done(P, st)) return mrc;
  TNX_CUDA(cudaStreamSynchronize(st));
  int m = std::min(done, (int)max_launches);
  for (int i = 0; i < m; ++i) {
    const Launch& L = P.slice_launches[i];
    types[i] = L.type == L_GATHER ? 0 : (L.type == L_SIMT || L.type == L_DOT || L.type == L_SIMTB) ? 1
             : (L.type == L_PACK || L.type == L_PERM) ? 2 : L.type == L_GEMM ? 3 : 4;
    vertices[i] = L.vertex;
    if (alg_bytes) {
      double b = 0.0;
      if (L.type == L_PERM) {
        const PermParams& pp = P.perms[L.idx];
        b = (double)pp.n_outer * pp.ts * (pp.mode == 0 ? 16.0 : pp.mode == 2 ? 32.0 : 24.0);
      } else if (L.type == L_PACK) {
        const PackParams& pk = P.packs[L.idx];
        b = (double)pk.rows * pk.K * 8.0 + (double)pk.rows * pk.kp * 4.0 * pk.nplanes;
      } else if (L.type == L_DOT) {
        b = (double)P.dots[L.idx].n * 16.0;
      }
      alg_bytes[i] = b;
    }
    float t = 0.f;
    TNX_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
    ms[i] = t;
  }
  for (auto& x : ev) cudaEventDestroy(x);
  *count = m;
  return TNX_OK;
}

int tnx_synchronize(void* plan) {
  Plan& P = *static_cast<Plan*>(plan);
  TNX_CUDA(cudaSetDevice(P.device));
  TNX_CUDA(cudaDeviceSynchronize());
  return TNX_OK;
}

int tnx_gemm_c64(const void* A, const void* B, void* C, int64_t batch, int64_t M, int64_t N,
                 int64_t K, int32_t precision, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char ebuf[256];
  if (gemm_init_attributes(ebuf, sizeof(ebuf))) return fail(TNX_ERR_CUDA, ebuf);
  const int64_t kp = align_up(K, 16);
  float *apl = nullptr, *bpl = nullptr;
  int splits = ((batch * M * N) % 2 == 0) ? gemm_choose_splits(batch, M, N, kp) : 1;
  const bool stack = precision == TNX_PREC_3XTF32 && gemm_use_stack(batch, M, N, kp, gemm_use_2sm(batch, M, N, kp, splits));
  TNX_CUDA(cudaMalloc(&apl, 16 * batch * M * kp));
  TNX_CUDA(cudaMalloc(&bpl, (stack ? 24 : 16) * batch * N * kp));
  auto simple = [&](IdxMap& m, int64_t rows, int64_t stride) {
    std::memset(&m, 0, sizeof(m));
    m.n = 1;
    m.dim[0] = rows;
    m.st0[0] = stride;
    m.lg[0] = -1;
  };
  PackParams pa{}, pb{};
  simple(pa.row, batch * M, K);
  simple(pa.col, K, 1);
  pa.src = static_cast<const float2*>(A);
  pa.dst = apl;
  pa.rows = batch * M;
  pa.K = K;
  pa.kp = kp;
  pa.plane_stride = pa.rows * kp;
  pa.nplanes = 4;
  pa.mix = precision == TNX_PREC_TF32_BF16X ? 1 : 0;
  simple(pb.row, batch * N, K);
  simple(pb.col, K, 1);
  pb.src = static_cast<const float2*>(B);
  pb.dst = bpl;
  pb.rows = batch * N;
  pb.K = K;
  pb.kp = kp;
  pb.plane_stride = pb.rows * kp;
  pb.nplanes = stack ? 6 : 4;
  pb.mix = precision == TNX_PREC_TF32_BF16X ? 2 : 0;
  cudaError_t e = launch_pack(pa, st);
  if (e == cudaSuccess) e = launch_pack(pb, st);
  if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
  GemmPlan g;
  float2* part = nullptr;
  if (splits > 1) TNX_CUDA(cudaMalloc(&part, 8 * (size_t)splits * batch * M * N));
  if (gemm_prepare(&g, apl, bpl, static_cast<float2*>(C), batch, M, N, kp, splits, part, ebuf, sizeof(ebuf),
                   stack ? 1 : 0))
    return fail(TNX_ERR_CUDA, ebuf);
  g.mix = precision == TNX_PREC_TF32_BF16X ? 1 : 0;
  e = launch_gemm(g, st);
  if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
  TNX_CUDA(cudaStreamSynchronize(st));
  cudaFree(apl);
  cudaFree(bpl);
  if (part) cudaFree(part);
  return TNX_OK;
}

int tnx_mma_peak(int32_t kind, int32_t cta_group, int64_t iters, void* stream, double* tflops,
                 double* sm_mhz, double* ms) {
  if (kind < 0 || kind > 2 || (cta_group != 1 && cta_group != 2) || iters < 8 || !tflops || !sm_mhz || !ms)
    return fail(TNX_ERR_INVALID, "tnx_mma_peak: kind 0 (tf32) / 1 (bf16) / 2 (ffma), cta_group 1 / 2, iters >= 8");
  char ebuf[256];
  if (gemm_mma_peak(kind, cta_group == 2, iters, static_cast<cudaStream_t>(stream), tflops, sm_mhz, ms, ebuf,
                    sizeof(ebuf)))
    return fail(TNX_ERR_CUDA, ebuf);
  return TNX_OK;
}

int tnx_clock_stamp(uint64_t* device_out, int32_t blocks, void* stream) {
  if (!device_out || blocks < 1) return fail(TNX_ERR_INVALID, "tnx_clock_stamp: need a device buffer of 3*blocks");
  cudaError_t e = launch_clock_stamp(reinterpret_cast<unsigned long long*>(device_out), blocks,
                                     static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(TNX_ERR_CUDA, cudaGetErrorString(e));
  return TNX_OK;
}

}  // extern "C"
