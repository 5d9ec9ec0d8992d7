// ApproxGraph index (IndexMode::ApproxGraph) on the GPU — SURVEY 8(f)#4.
//
// The reference builds a hierarchical navigable-small-world graph by
// sequential insertion (nn_index.cpp:83-237: seeded levels, greedy descent,
// beam search per layer, links pruned to the closest cap) and answers graph
// queries by greedy descent plus a beam search on layer 0 (:288-333, :351-366),
// falling back to a scan when fewer than k neighbours come back. Insertion is
// inherently sequential (each node searches the graph built so far), so this
// is a replacement, not a replay:
//
//  * levels: the reference's generator exactly (splitmix64 stream of
//    seed ^ 0xa02bdbf7bb3c0a7, level = floor(-ln(u) / ln M)), so the layer
//    populations, the maximum level and the entry point (the first node to
//    reach it) are the reference's;
//  * links: every node's cap nearest neighbours among the nodes of that layer
//    (2M on layer 0, M above), found by the exact kNN kernels of this library
//    (cell grid for d <= 3, tcgen05 filter for d >= 4): one batched exact
//    search per layer instead of n sequential beam searches;
//  * queries: one warp per query runs the reference's algorithm — greedy
//    descent on the upper layers (lexicographic (dist_sq, index) moves,
//    :139-161) and the bounded best-first search on layer 0 with beam
//    max(64, 2k) (or query_beam), visited nodes in a per-warp hash table in
//    shared memory, the result list sorted by (dist_sq, index) in registers;
//    fewer than k results after the exclusion falls back to the exact scan,
//    as the reference does (:311-329). dist_sq is the reference's key.
//
// Graphs serialize in the reference's layout (nn_index.cpp:397-416), and a
// reference-written graph loads (fmgp_graph_load) and is searched here.
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "capi_common.h"
#include "capi_model.h"
#include "fmgp_common.cuh"
#include "fmgp_internal.h"
#include "../../include/fmgp_b200.h"

using namespace fmgp_capi;

struct fmgp_graph {
  const fmgp_index* ix = nullptr;  // searched points (the caller keeps the index alive while the graph is used)
  int device = 0;                  // the index's device, kept so destroy never reads the index
  int32_t max_degree = 16, build_beam = 100, query_beam = 0;
  uint64_t seed = 0;
  int32_t entry = 0, max_level = 0;
  int32_t w0 = 0, w1 = 0;          // widths of the layer-0 / upper-layer link rows
  int32_t* levels = nullptr;       // n
  int32_t* links0 = nullptr;       // n x w0, -1 padded
  int32_t* up_base = nullptr;      // n: first upper-layer record of node i (records of a node: layers 1..level)
  int32_t* up = nullptr;           // records of (w1 + 1) ints: count, ids (-1 padded)
  int64_t up_records = 0;
};

namespace fmgp {
namespace {

constexpr int kGWarps = 4;          // warps per CTA of the search kernel
constexpr int kHashBits = 12;       // visited table: 4096 slots per warp
constexpr int kHashProbe = 32;

__device__ __forceinline__ uint64_t splitmix_at(uint64_t s0, int64_t i) {
  // output i of the reference's splitmix64 stream (the state advances by the
  // golden increment per call, nn_index.cpp:44-49)
  uint64_t z = s0 + static_cast<uint64_t>(i + 1) * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void levels_kernel(int64_t n, uint64_t s0, double ml, int32_t* __restrict__ levels,
                              int32_t* __restrict__ maxlvl) {
  int32_t mx = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t z = splitmix_at(s0, i);
    const double u = __dadd_rn(__dmul_rn(static_cast<double>(z >> 11), 0x1p-53), 0x1p-54);  // assign_level :84
    const int lvl = static_cast<int>(__dmul_rn(-log(u), ml));
    levels[i] = lvl;
    mx = max(mx, lvl);
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxlvl, mx);
}

__global__ void entry_kernel(int64_t n, const int32_t* __restrict__ levels, const int32_t* __restrict__ maxlvl,
                             int32_t* __restrict__ entry) {
  const int32_t mx = *maxlvl;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (levels[i] == mx) atomicMin(entry, static_cast<int32_t>(i));  // the first node to reach it (:231-234)
}

// Exclusive scan of int32 values (single CTA, chunked per thread; index-build metadata only).
__global__ void scan1_kernel(const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                             int32_t* __restrict__ total) {
  __shared__ int32_t part[1024];
  const int t = threadIdx.x, T = blockDim.x;
  const int64_t per = (n + T - 1) / T, b = t * per, e = n < b + per ? n : b + per;
  int32_t s = 0;
  for (int64_t i = b; i < e; ++i) s += in[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int32_t acc = 0;
    for (int q = 0; q < T; ++q) {
      const int32_t v = part[q];
      part[q] = acc;
      acc += v;
    }
    if (total) *total = acc;
  }
  __syncthreads();
  int32_t acc = part[t];
  for (int64_t i = b; i < e; ++i) {
    const int32_t v = in[i];
    out[i] = acc;
    acc += v;
  }
}

__global__ void flag_level_kernel(int64_t n, const int32_t* __restrict__ levels, int L, int32_t* __restrict__ flag) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    flag[i] = levels[i] >= L ? 1 : 0;
}

__global__ void compact_kernel(int64_t n, const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                               const double* __restrict__ P, int d, int32_t* __restrict__ ids,
                               double* __restrict__ PL) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!flag[i]) continue;
    const int64_t r = pos[i];
    ids[r] = static_cast<int32_t>(i);
    for (int t = 0; t < d; ++t) PL[r * d + t] = P[i * d + t];
  }
}

// Layer-0 rows: the kk nearest (self excluded) as links, -1 padded to w0.
__global__ void links0_kernel(int64_t n, const int32_t* __restrict__ nn, int kk, int w0, int32_t* __restrict__ links0) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * w0;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / w0;
    const int t = static_cast<int>(e - i * w0);
    links0[e] = t < kk ? nn[i * kk + t] : -1;
  }
}

// Upper layer L: record (up_base[node] + L - 1) = count, then the node ids of
// its kk nearest among the layer's nodes (subset indices mapped back).
__global__ void links_up_kernel(int64_t nl, const int32_t* __restrict__ ids, const int32_t* __restrict__ nn, int kk,
                                int L, int w1, const int32_t* __restrict__ up_base, int32_t* __restrict__ up) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < nl;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t node = ids[r];
    int32_t* rec = up + (static_cast<int64_t>(up_base[node]) + L - 1) * (w1 + 1);
    rec[0] = kk;
    for (int t = 0; t < w1; ++t) rec[1 + t] = t < kk ? ids[nn[r * kk + t]] : -1;
  }
}

unsigned g1d(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 4096) b = 4096;
  return static_cast<unsigned>(b);
}

// ---------------------------------------------------------------- search

struct GCand {
  double d;
  int32_t i;  // bit 31: expanded
};

__device__ __forceinline__ bool gless(const GCand& a, const GCand& b) {
  const int32_t ia = a.i & 0x7fffffff, ib = b.i & 0x7fffffff;
  return a.d < b.d || (a.d == b.d && ia < ib);
}
__device__ __forceinline__ GCand gshfl(const GCand& c, int src) {
  return GCand{__shfl_sync(0xffffffffu, c.d, src), __shfl_sync(0xffffffffu, c.i, src)};
}
__device__ __forceinline__ GCand gshfl_xor(const GCand& c, int m) {
  return GCand{__shfl_xor_sync(0xffffffffu, c.d, m), __shfl_xor_sync(0xffffffffu, c.i, m)};
}
__device__ __forceinline__ GCand gcx(GCand v, int stride, bool up, int lane) {
  const GCand o = gshfl_xor(v, stride);
  const bool lower = (lane & stride) == 0;
  return ((lower == up) == gless(o, v)) ? o : v;
}
__device__ __forceinline__ GCand gsort32(GCand v, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) v = gcx(v, stride, (lane & size) == 0, lane);
  return v;
}
__device__ __forceinline__ GCand gclean32(GCand v, int lane) {
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) v = gcx(v, stride, true, lane);
  return v;
}
__device__ __forceinline__ void gmerge32(GCand& a, GCand& b, int lane) {
  const GCand br = gshfl(b, 31 - lane);
  const GCand lo = gless(br, a) ? br : a;
  const GCand hi = gless(br, a) ? a : br;
  a = gclean32(lo, lane);
  b = gclean32(hi, lane);
}

// Keep the 32E smallest of (list u batch), list ascending over (e, lane).
template <int E>
__device__ __forceinline__ void gmerge_batch(GCand (&Lst)[E], GCand c, int lane) {
  c = gsort32(c, lane);
  const GCand cr = gshfl(c, 31 - lane);
  GCand x = gless(cr, Lst[E - 1]) ? cr : Lst[E - 1];
  x = gclean32(x, lane);
#pragma unroll
  for (int e = E - 1; e >= 1; --e) {
    GCand a = Lst[e - 1];
    GCand b = (e == E - 1) ? x : Lst[e];
    gmerge32(a, b, lane);
    Lst[e - 1] = a;
    Lst[e] = b;
  }
  if (E == 1) Lst[0] = x;
}

struct GraphView {
  const double* P;
  int32_t n, d;
  int32_t entry, max_level, w0, w1;
  const int32_t* links0;
  const int32_t* up_base;
  const int32_t* up;
};

__device__ __forceinline__ double gdist(const double* q, const double* P, int d, int32_t j) {
  return dist_sq_dyn(q, P + static_cast<int64_t>(j) * d, d);
}

// Visited test-and-set in the warp's table; false = first visit. A full probe
// window reports "not visited" (the node is evaluated again; the list merge
// drops exact duplicates).
__device__ __forceinline__ bool visited_tas(int32_t* ht, int32_t u) {
  uint32_t h = (static_cast<uint32_t>(u) * 0x9E3779B1u) >> (32 - kHashBits);
  for (int p = 0; p < kHashProbe; ++p) {
    const uint32_t s = (h + p) & ((1u << kHashBits) - 1);
    const int32_t cur = ht[s];
    if (cur == u) return true;
    if (cur == -1) {
      const int32_t old = atomicCAS(&ht[s], -1, u);
      if (old == -1) return false;
      if (old == u) return true;
    }
  }
  return false;
}

// One warp per query: greedy descent (nn_index.cpp:139-161), then the bounded
// best-first search on layer 0 (:90-137) with a list of `beam` (<= 32 E)
// entries. Writes the first k entries whose index is not `exclude`; a query
// with fewer than k is flagged for the exact fallback (:311-329).
template <int E>
__global__ void __launch_bounds__(kGWarps * 32)
graph_search_kernel(GraphView g, const double* __restrict__ Q, int64_t nq, int k, int beam,
                    const int32_t* __restrict__ excl, int32_t* __restrict__ out_i, double* __restrict__ out_d,
                    int32_t* __restrict__ short_flag, unsigned long long* __restrict__ evals) {
  extern __shared__ int32_t s_ht[];  // kGWarps visited tables of 2^kHashBits slots
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int32_t* ht = s_ht + (wib << kHashBits);
  unsigned long long my_evals = 0;
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * kGWarps + wib; w < nq;
       w += static_cast<int64_t>(gridDim.x) * kGWarps) {
    const double* q = Q + w * g.d;
    for (int s = lane; s < (1 << kHashBits); s += 32) ht[s] = -1;
    __syncwarp();
    // greedy descent: the running (dist, index) minimum over each visited link list
    int32_t cur = g.entry;
    double best = gdist(q, g.P, g.d, cur);
    my_evals += (lane == 0);
    for (int L = g.max_level; L >= 1; --L) {
      while (true) {
        const int32_t* rec = g.up + (static_cast<int64_t>(g.up_base[cur]) + L - 1) * (g.w1 + 1);
        const int cnt = rec[0];
        GCand m{best, cur};
        for (int t0 = 0; t0 < cnt; t0 += 32) {
          GCand c{INFINITY, INT_MAX};
          if (t0 + lane < cnt) {
            const int32_t u = rec[1 + t0 + lane];
            c = GCand{gdist(q, g.P, g.d, u), u};
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const GCand x = gshfl_xor(c, o);
            if (gless(x, c)) c = x;
          }
          if (gless(c, m)) m = c;
        }
        my_evals += (lane == 0) ? cnt : 0;
        if (m.i == cur) break;
        cur = m.i;
        best = m.d;
      }
    }
    // layer 0
    GCand Lst[E];
#pragma unroll
    for (int e = 0; e < E; ++e) Lst[e] = GCand{INFINITY, INT_MAX};
    if (lane == 0) Lst[0] = GCand{best, cur};
    if (lane == 0) ht[(static_cast<uint32_t>(cur) * 0x9E3779B1u) >> (32 - kHashBits)] = cur;
    __syncwarp();
    while (true) {
      // the closest entry not yet expanded
      int pick_e = -1, pick_l = 0;
#pragma unroll
      for (int e = E - 1; e >= 0; --e) {
        const bool open = (Lst[e].i & 0x80000000) == 0 && Lst[e].i != INT_MAX && (32 * e + lane) < beam;
        const unsigned bal = __ballot_sync(0xffffffffu, open);
        if (bal) {
          pick_e = e;
          pick_l = __ffs(bal) - 1;
        }
      }
      if (pick_e < 0) break;
      int32_t c = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e == pick_e) {
          c = __shfl_sync(0xffffffffu, Lst[e].i, pick_l);
          if (lane == pick_l) Lst[e].i |= static_cast<int32_t>(0x80000000u);
        }
      }
      const int32_t* row = g.links0 + static_cast<int64_t>(c) * g.w0;
      for (int t0 = 0; t0 < g.w0; t0 += 32) {
        GCand cand{INFINITY, INT_MAX};
        const int32_t u = t0 + lane < g.w0 ? row[t0 + lane] : -1;
        bool fresh = false;
        if (u >= 0) fresh = !visited_tas(ht, u);
        if (fresh) cand = GCand{gdist(q, g.P, g.d, u), u};
        my_evals += fresh ? 1 : 0;
        GCand worst = gshfl(Lst[E - 1], 31);
        if (beam < 32 * E) {
          const int wpos = beam - 1;
#pragma unroll
          for (int e = 0; e < E; ++e)
            if (e == wpos / 32) worst = gshfl(Lst[e], wpos & 31);
        }
        const bool pass = fresh && gless(cand, worst);
        if (!__any_sync(0xffffffffu, pass)) continue;
        if (!pass) cand = GCand{INFINITY, INT_MAX};
        gmerge_batch<E>(Lst, cand, lane);
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (32 * e + lane >= beam) Lst[e] = GCand{INFINITY, INT_MAX};
      }
    }
    // drop exact duplicates (a hash-overflow re-visit) and the excluded index, write k
    const int32_t ex = excl != nullptr ? excl[w] : -1;
    int written = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const GCand c = Lst[e];
      const int32_t id = c.i & 0x7fffffff;
      const GCand prev = GCand{__shfl_up_sync(0xffffffffu, c.d, 1), __shfl_up_sync(0xffffffffu, c.i, 1)};
      GCand prev_e = prev;
      if (e > 0) {
        const GCand last = gshfl(Lst[e > 0 ? e - 1 : 0], 31);
        if (lane == 0) prev_e = last;
      }
      const bool dupe = (e > 0 || lane > 0) && prev_e.d == c.d && (prev_e.i & 0x7fffffff) == id;
      const bool keep = id != INT_MAX && id != ex && !dupe && (32 * e + lane) < beam;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      const int pos = written + __popc(bal & ((1u << lane) - 1));
      if (keep && pos < k) {
        out_i[w * k + pos] = id;
        if (out_d) out_d[w * k + pos] = sqrt(c.d);
      }
      written += __popc(bal);
    }
    if (lane == 0) short_flag[w] = written < k ? 1 : 0;
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) my_evals += __shfl_xor_sync(0xffffffffu, my_evals, o);
  if (lane == 0 && evals != nullptr) atomicAdd(evals, my_evals);
}

GraphView view_of(const fmgp_graph* g) {
  return GraphView{g->ix->P, static_cast<int32_t>(g->ix->n), g->ix->d, g->entry, g->max_level, g->w0, g->w1,
                   g->links0, g->up_base, g->up};
}

cudaError_t launch_search(const fmgp_graph* g, const double* dQ, int64_t nq, int k, int beam, const int32_t* dE,
                          int32_t* dI, double* dD, int32_t* dShort, unsigned long long* dEv, cudaStream_t s) {
  const GraphView v = view_of(g);
  const int sms = num_sms_current();
  int64_t blocks = (nq + kGWarps - 1) / kGWarps;
  if (blocks > static_cast<int64_t>(sms) * 8) blocks = static_cast<int64_t>(sms) * 8;
  const unsigned nb = static_cast<unsigned>(blocks < 1 ? 1 : blocks);
  const int smem = static_cast<int>(sizeof(int32_t) * kGWarps << kHashBits);
  cudaError_t e;
  if (beam <= 32) {
    e = cudaFuncSetAttribute(graph_search_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      graph_search_kernel<1><<<nb, kGWarps * 32, smem, s>>>(v, dQ, nq, k, beam, dE, dI, dD, dShort, dEv);
  } else if (beam <= 64) {
    e = cudaFuncSetAttribute(graph_search_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      graph_search_kernel<2><<<nb, kGWarps * 32, smem, s>>>(v, dQ, nq, k, beam, dE, dI, dD, dShort, dEv);
  } else {
    e = cudaFuncSetAttribute(graph_search_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess)
      graph_search_kernel<4><<<nb, kGWarps * 32, smem, s>>>(v, dQ, nq, k, beam, dE, dI, dD, dShort, dEv);
  }
  if (e != cudaSuccess) return e;
  note_launches(1);
  return cudaGetLastError();
}

constexpr int kMaxBeam = 128;  // list capacity of the search kernel; larger beams search exactly

}  // namespace
}  // namespace fmgp

using fmgp::g1d;

namespace {

void graph_free(fmgp_graph* g) {
  if (g == nullptr) return;
  for (void* p : {static_cast<void*>(g->levels), static_cast<void*>(g->links0), static_cast<void*>(g->up_base),
                  static_cast<void*>(g->up)})
    if (p) cudaFree(p);
  delete g;
}

// up_base = exclusive scan of levels; allocates up (records x (w1 + 1)).
cudaError_t alloc_upper(fmgp_graph* g, int64_t n, cudaStream_t s) {
  int32_t* tot = nullptr;
  cudaError_t e = cudaMalloc(&g->up_base, sizeof(int32_t) * n);
  if (e == cudaSuccess) e = cudaMalloc(&tot, sizeof(int32_t));
  if (e == cudaSuccess) {
    fmgp::scan1_kernel<<<1, 1024, 0, s>>>(g->levels, n, g->up_base, tot);
    int32_t h = 0;
    e = cudaMemcpyAsync(&h, tot, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    g->up_records = h;
  }
  if (tot) cudaFree(tot);
  if (e == cudaSuccess) e = cudaMalloc(&g->up, sizeof(int32_t) * (g->up_records > 0 ? g->up_records : 1) * (g->w1 + 1));
  if (e == cudaSuccess && g->up_records > 0)
    e = cudaMemsetAsync(g->up, 0, sizeof(int32_t) * g->up_records * (g->w1 + 1), s);
  return e;
}

}  // namespace

extern "C" {

int fmgp_graph_build(const fmgp_index* ix, int32_t max_degree, int32_t build_beam, int32_t query_beam,
                     uint64_t seed, fmgp_graph** out) {
  if (out == nullptr || ix == nullptr) return fail(FMGP_EINVAL, "graph: null argument");
  *out = nullptr;
  if (max_degree < 2 || build_beam < 1) return fail(FMGP_EINVAL, "NeighborIndex: invalid graph parameters");
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(ix->device));
  Stream st;
  FMGP_CUDA(st.create());
  auto* g = new fmgp_graph();
  g->ix = ix;
  g->device = ix->device;
  g->max_degree = max_degree;
  g->build_beam = build_beam;
  g->query_beam = query_beam;
  g->seed = seed;
  const int64_t n = ix->n;
  const int d = ix->d;
  g->w0 = 2 * max_degree;
  g->w1 = max_degree;
  const int sms = num_sms_current();
  cudaError_t e = cudaMalloc(&g->levels, sizeof(int32_t) * n);
  int32_t* dmx = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&dmx, sizeof(int32_t) * 2);
  if (e == cudaSuccess) {
    const int32_t init[2] = {0, INT32_MAX};
    e = cudaMemcpyAsync(dmx, init, sizeof(init), cudaMemcpyHostToDevice, st.s);
  }
  if (e == cudaSuccess) {
    const double ml = 1.0 / std::log(static_cast<double>(max_degree));
    fmgp::levels_kernel<<<g1d(n), 256, 0, st.s>>>(n, seed ^ 0xa02bdbf7bb3c0a7ULL, ml, g->levels, dmx);
    fmgp::entry_kernel<<<g1d(n), 256, 0, st.s>>>(n, g->levels, dmx, dmx + 1);
    fmgp::note_launches(2);
    int32_t h[2];
    e = cudaMemcpyAsync(h, dmx, sizeof(h), cudaMemcpyDeviceToHost, st.s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st.s);
    g->max_level = h[0];
    g->entry = h[1];
  }
  if (dmx) cudaFree(dmx);
  // layer 0: the 2M nearest of every node
  if (e == cudaSuccess) e = cudaMalloc(&g->links0, sizeof(int32_t) * n * g->w0);
  const int k0 = static_cast<int>(std::min<int64_t>(g->w0, n - 1));
  if (e == cudaSuccess && k0 > 0) {
    DevBuf<int32_t> nn;
    e = nn.alloc(static_cast<size_t>(n) * k0, st.s);
    if (e == cudaSuccess) e = fmgp::knn_exact(ix->P, n, ix->P, n, d, k0, 0, nullptr, 0, nn.p, nullptr, sms, st.s);
    if (e == cudaSuccess) {
      fmgp::links0_kernel<<<g1d(n * g->w0), 256, 0, st.s>>>(n, nn.p, k0, g->w0, g->links0);
      fmgp::note_launches(1);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st.s);
  } else if (e == cudaSuccess) {
    e = cudaMemsetAsync(g->links0, 0xFF, sizeof(int32_t) * n * g->w0, st.s);
  }
  if (e == cudaSuccess) e = alloc_upper(g, n, st.s);
  // upper layers: the M nearest among the layer's nodes
  for (int L = 1; e == cudaSuccess && L <= g->max_level; ++L) {
    DevBuf<int32_t> flag, pos, ids, nn, tot;
    DevBuf<double> PL;
    e = flag.alloc(n, st.s);
    if (e == cudaSuccess) e = pos.alloc(n, st.s);
    if (e == cudaSuccess) e = tot.alloc(1, st.s);
    if (e != cudaSuccess) break;
    fmgp::flag_level_kernel<<<g1d(n), 256, 0, st.s>>>(n, g->levels, L, flag.p);
    fmgp::scan1_kernel<<<1, 1024, 0, st.s>>>(flag.p, n, pos.p, tot.p);
    fmgp::note_launches(2);
    int32_t nl = 0;
    e = cudaMemcpyAsync(&nl, tot.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st.s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st.s);
    if (e != cudaSuccess || nl < 1) break;
    e = ids.alloc(nl, st.s);
    if (e == cudaSuccess) e = PL.alloc(static_cast<size_t>(nl) * d, st.s);
    if (e != cudaSuccess) break;
    fmgp::compact_kernel<<<g1d(n), 256, 0, st.s>>>(n, flag.p, pos.p, ix->P, d, ids.p, PL.p);
    fmgp::note_launches(1);
    const int kl = std::min(g->w1, nl - 1);
    if (kl > 0) {
      e = nn.alloc(static_cast<size_t>(nl) * kl, st.s);
      if (e == cudaSuccess) e = fmgp::knn_exact(PL.p, nl, PL.p, nl, d, kl, 0, nullptr, 0, nn.p, nullptr, sms, st.s);
    }
    if (e == cudaSuccess) {
      fmgp::links_up_kernel<<<g1d(nl), 256, 0, st.s>>>(nl, ids.p, nn.p, kl, L, g->w1, g->up_base, g->up);
      fmgp::note_launches(1);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st.s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st.s);
  if (e != cudaSuccess) {
    graph_free(g);
    return cuda_fail(e, "fmgp_graph_build");
  }
  *out = g;
  return FMGP_OK;
}

int fmgp_graph_load(const fmgp_index* ix, int32_t max_degree, int32_t build_beam, int32_t query_beam, uint64_t seed,
                    int32_t entry, int32_t max_level, const int32_t* levels, const uint32_t* counts,
                    const int32_t* ids, fmgp_graph** out) {
  if (out == nullptr || ix == nullptr || levels == nullptr || counts == nullptr)
    return fail(FMGP_EINVAL, "graph: null argument");
  *out = nullptr;
  const int64_t n = ix->n;
  if (entry < 0 || entry >= n) return fail(FMGP_EINVAL, "neighbor-index entry point out of range");
  // widths and layout from the serialized counts (node-major, layer 0 first)
  uint32_t w0 = 0, w1 = 0;
  int64_t c = 0, total_ids = 0;
  std::vector<int32_t> base(n);
  int64_t rec = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (levels[i] < 0) return fail(FMGP_EINVAL, "negative node level in neighbor index");
    base[i] = static_cast<int32_t>(rec);
    for (int l = 0; l <= levels[i]; ++l) {
      const uint32_t cnt = counts[c++];
      (l == 0 ? w0 : w1) = std::max(l == 0 ? w0 : w1, cnt);
      total_ids += cnt;
    }
    rec += levels[i];
  }
  for (int64_t t = 0; t < total_ids; ++t)
    if (ids[t] < 0 || ids[t] >= n) return fail(FMGP_EINVAL, "neighbor id out of range");
  std::vector<int32_t> l0(static_cast<size_t>(n) * std::max<uint32_t>(w0, 1), -1);
  std::vector<int32_t> upv(static_cast<size_t>(std::max<int64_t>(rec, 1)) * (w1 + 1), -1);
  c = 0;
  int64_t p = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int l = 0; l <= levels[i]; ++l) {
      const uint32_t cnt = counts[c++];
      if (l == 0) {
        for (uint32_t t = 0; t < cnt; ++t) l0[static_cast<size_t>(i) * w0 + t] = ids[p + t];
      } else {
        int32_t* r = upv.data() + (static_cast<size_t>(base[i]) + l - 1) * (w1 + 1);
        r[0] = static_cast<int32_t>(cnt);
        for (uint32_t t = 0; t < cnt; ++t) r[1 + t] = ids[p + t];
      }
      p += cnt;
    }
  }
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(ix->device));
  auto* g = new fmgp_graph();
  g->ix = ix;
  g->device = ix->device;
  g->max_degree = max_degree;
  g->build_beam = build_beam;
  g->query_beam = query_beam;
  g->seed = seed;
  g->entry = entry;
  g->max_level = max_level;
  g->w0 = static_cast<int32_t>(std::max<uint32_t>(w0, 1));
  g->w1 = static_cast<int32_t>(w1);
  g->up_records = rec;
  cudaError_t e = cudaMalloc(&g->levels, sizeof(int32_t) * n);
  if (e == cudaSuccess) e = cudaMemcpy(g->levels, levels, sizeof(int32_t) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&g->links0, sizeof(int32_t) * l0.size());
  if (e == cudaSuccess) e = cudaMemcpy(g->links0, l0.data(), sizeof(int32_t) * l0.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&g->up_base, sizeof(int32_t) * n);
  if (e == cudaSuccess) e = cudaMemcpy(g->up_base, base.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&g->up, sizeof(int32_t) * upv.size());
  if (e == cudaSuccess) e = cudaMemcpy(g->up, upv.data(), sizeof(int32_t) * upv.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    graph_free(g);
    return cuda_fail(e, "fmgp_graph_load");
  }
  *out = g;
  return FMGP_OK;
}

int fmgp_graph_info(const fmgp_graph* g, int32_t* entry, int32_t* max_level, int64_t* counts_total,
                    int64_t* ids_total) {
  if (g == nullptr) return fail(FMGP_EINVAL, "null graph");
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(g->ix->device));
  const int64_t n = g->ix->n;
  std::vector<int32_t> lv(n), l0(static_cast<size_t>(n) * g->w0);
  std::vector<int32_t> upv(static_cast<size_t>(std::max<int64_t>(g->up_records, 1)) * (g->w1 + 1));
  FMGP_CUDA(cudaMemcpy(lv.data(), g->levels, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  FMGP_CUDA(cudaMemcpy(l0.data(), g->links0, sizeof(int32_t) * l0.size(), cudaMemcpyDeviceToHost));
  if (g->up_records > 0)
    FMGP_CUDA(cudaMemcpy(upv.data(), g->up, sizeof(int32_t) * g->up_records * (g->w1 + 1), cudaMemcpyDeviceToHost));
  int64_t ct = 0, it = 0;
  for (int64_t i = 0; i < n; ++i) {
    ct += 1 + lv[i];
    for (int t = 0; t < g->w0; ++t) it += l0[static_cast<size_t>(i) * g->w0 + t] >= 0;
  }
  for (int64_t r = 0; r < g->up_records; ++r) it += upv[static_cast<size_t>(r) * (g->w1 + 1)];
  if (entry) *entry = g->entry;
  if (max_level) *max_level = g->max_level;
  if (counts_total) *counts_total = ct;
  if (ids_total) *ids_total = it;
  return FMGP_OK;
}

int fmgp_graph_export(const fmgp_graph* g, int32_t* levels, uint32_t* counts, int32_t* ids) {
  if (g == nullptr || levels == nullptr || counts == nullptr || ids == nullptr) return fail(FMGP_EINVAL, "null argument");
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(g->ix->device));
  const int64_t n = g->ix->n;
  std::vector<int32_t> l0(static_cast<size_t>(n) * g->w0), base(n);
  std::vector<int32_t> upv(static_cast<size_t>(std::max<int64_t>(g->up_records, 1)) * (g->w1 + 1));
  FMGP_CUDA(cudaMemcpy(levels, g->levels, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  FMGP_CUDA(cudaMemcpy(l0.data(), g->links0, sizeof(int32_t) * l0.size(), cudaMemcpyDeviceToHost));
  FMGP_CUDA(cudaMemcpy(base.data(), g->up_base, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  if (g->up_records > 0)
    FMGP_CUDA(cudaMemcpy(upv.data(), g->up, sizeof(int32_t) * g->up_records * (g->w1 + 1), cudaMemcpyDeviceToHost));
  int64_t c = 0, p = 0;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t cnt = 0;
    for (int t = 0; t < g->w0; ++t) {
      const int32_t u = l0[static_cast<size_t>(i) * g->w0 + t];
      if (u >= 0) ids[p + cnt++] = u;
    }
    counts[c++] = cnt;
    p += cnt;
    for (int l = 1; l <= levels[i]; ++l) {
      const int32_t* r = upv.data() + (static_cast<size_t>(base[i]) + l - 1) * (g->w1 + 1);
      counts[c++] = static_cast<uint32_t>(r[0]);
      for (int t = 0; t < r[0]; ++t) ids[p + t] = r[1 + t];
      p += r[0];
    }
  }
  return FMGP_OK;
}

// Shared driver of the two query entry points: graph search, then the exact
// search for the queries that came back short (and for beams above the
// kernel's list capacity).
static int graph_query(const fmgp_graph* g, const double* Q, int64_t nq, int32_t k, int32_t beam,
                       const int32_t* exclude, int32_t* idx_out, double* dist_out, uint64_t* dist_evals) {
  const fmgp_index* ix = g->ix;
  if (nq <= 0) return FMGP_OK;
  if (!all_finite(Q, nq * ix->d)) return fail(FMGP_EINVAL, "query_knn: non-finite query");
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(ix->device));
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dQ, dD;
  DevBuf<int32_t> dI, dE, dShort;
  DevBuf<unsigned long long> dEv;
  FMGP_CUDA(dQ.alloc(static_cast<size_t>(nq) * ix->d, st.s));
  FMGP_CUDA(dI.alloc(static_cast<size_t>(nq) * k, st.s));
  FMGP_CUDA(dD.alloc(static_cast<size_t>(nq) * k, st.s));
  FMGP_CUDA(dShort.alloc(nq, st.s));
  FMGP_CUDA(dEv.alloc(1, st.s));
  FMGP_CUDA(cudaMemsetAsync(dEv.p, 0, sizeof(unsigned long long), st.s));
  FMGP_CUDA(cudaMemcpyAsync(dQ.p, Q, sizeof(double) * nq * ix->d, cudaMemcpyHostToDevice, st.s));
  if (exclude != nullptr) {
    FMGP_CUDA(dE.alloc(nq, st.s));
    FMGP_CUDA(cudaMemcpyAsync(dE.p, exclude, sizeof(int32_t) * nq, cudaMemcpyHostToDevice, st.s));
  }
  std::vector<int32_t> shortq(nq, 1);
  uint64_t ev = 0;
  if (beam <= fmgp::kMaxBeam) {
    FMGP_CUDA(fmgp::launch_search(g, dQ.p, nq, k, beam, dE.p, dI.p, dD.p, dShort.p, dEv.p, st.s));
    FMGP_CUDA(cudaMemcpyAsync(shortq.data(), dShort.p, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st.s));
    unsigned long long h = 0;
    FMGP_CUDA(cudaMemcpyAsync(&h, dEv.p, sizeof(h), cudaMemcpyDeviceToHost, st.s));
    FMGP_CUDA(cudaStreamSynchronize(st.s));
    ev = h;
  }
  // exact fallback for the short queries (the reference's scan, nn_index.cpp:311-329)
  std::vector<int32_t> rows;
  for (int64_t q = 0; q < nq; ++q)
    if (shortq[q]) rows.push_back(static_cast<int32_t>(q));
  if (!rows.empty()) {
    const int64_t nr = static_cast<int64_t>(rows.size());
    std::vector<double> qh(static_cast<size_t>(nr) * ix->d);
    std::vector<int32_t> eh(nr, -1);
    for (int64_t r = 0; r < nr; ++r) {
      std::memcpy(qh.data() + r * ix->d, Q + static_cast<int64_t>(rows[r]) * ix->d, sizeof(double) * ix->d);
      if (exclude) eh[r] = exclude[rows[r]];
      ev += static_cast<uint64_t>(ix->n) - (eh[r] >= 0 && eh[r] < ix->n ? 1 : 0);
    }
    DevBuf<double> fQ, fD;
    DevBuf<int32_t> fI, fE;
    FMGP_CUDA(fQ.alloc(qh.size(), st.s));
    FMGP_CUDA(fE.alloc(nr, st.s));
    FMGP_CUDA(fI.alloc(static_cast<size_t>(nr) * k, st.s));
    FMGP_CUDA(fD.alloc(static_cast<size_t>(nr) * k, st.s));
    FMGP_CUDA(cudaMemcpyAsync(fQ.p, qh.data(), sizeof(double) * qh.size(), cudaMemcpyHostToDevice, st.s));
    FMGP_CUDA(cudaMemcpyAsync(fE.p, eh.data(), sizeof(int32_t) * nr, cudaMemcpyHostToDevice, st.s));
    FMGP_CUDA(fmgp::knn_exact(fQ.p, nr, ix->P, ix->n, ix->d, k, -1, fE.p, 0, fI.p, fD.p, num_sms_current(), st.s));
    FMGP_CUDA(fmgp::sqrt_inplace_launch(fD.p, nr * k, st.s));
    std::vector<int32_t> ih(static_cast<size_t>(nr) * k);
    std::vector<double> dh(static_cast<size_t>(nr) * k);
    FMGP_CUDA(cudaMemcpyAsync(ih.data(), fI.p, sizeof(int32_t) * ih.size(), cudaMemcpyDeviceToHost, st.s));
    FMGP_CUDA(cudaMemcpyAsync(dh.data(), fD.p, sizeof(double) * dh.size(), cudaMemcpyDeviceToHost, st.s));
    if (idx_out) FMGP_CUDA(cudaMemcpyAsync(idx_out, dI.p, sizeof(int32_t) * nq * k, cudaMemcpyDeviceToHost, st.s));
    if (dist_out) FMGP_CUDA(cudaMemcpyAsync(dist_out, dD.p, sizeof(double) * nq * k, cudaMemcpyDeviceToHost, st.s));
    FMGP_CUDA(cudaStreamSynchronize(st.s));
    for (int64_t r = 0; r < nr; ++r) {
      const int64_t q = rows[r];
      std::memcpy(idx_out + q * k, ih.data() + r * k, sizeof(int32_t) * k);
      if (dist_out) std::memcpy(dist_out + q * k, dh.data() + r * k, sizeof(double) * k);
    }
  } else {
    FMGP_CUDA(cudaMemcpyAsync(idx_out, dI.p, sizeof(int32_t) * nq * k, cudaMemcpyDeviceToHost, st.s));
    if (dist_out) FMGP_CUDA(cudaMemcpyAsync(dist_out, dD.p, sizeof(double) * nq * k, cudaMemcpyDeviceToHost, st.s));
    FMGP_CUDA(cudaStreamSynchronize(st.s));
  }
  if (dist_evals) *dist_evals += ev;
  return FMGP_OK;
}

int fmgp_graph_query_knn(const fmgp_graph* g, const double* Q, int64_t nq, int32_t k, const int32_t* exclude,
                         int32_t* idx_out, double* dist_out, uint64_t* dist_evals) {
  if (g == nullptr || idx_out == nullptr) return fail(FMGP_EINVAL, "graph: null argument");
  bool any_excl = false;
  if (exclude != nullptr)
    for (int64_t q = 0; q < nq; ++q) any_excl |= exclude[q] >= 0;
  if (k < 1 || k > g->ix->n - (any_excl ? 1 : 0)) return fail(FMGP_EINVAL, "query_knn: k out of range");
  // beam (nn_index.cpp:302-305): query_beam or max(64, 2k), at least k (+1 with an exclusion)
  int beam = g->query_beam > 0 ? g->query_beam : std::max(64, 2 * k);
  beam = std::max(beam, k + (any_excl ? 1 : 0));
  return graph_query(g, Q, nq, k, beam, exclude, idx_out, dist_out, dist_evals);
}

int fmgp_graph_nearest(const fmgp_graph* g, const double* Q, int64_t nq, int32_t* idx_out, uint64_t* dist_evals) {
  if (g == nullptr || idx_out == nullptr) return fail(FMGP_EINVAL, "graph: null argument");
  const int beam = g->query_beam > 0 ? g->query_beam : 64;  // nn_index.cpp:363
  return graph_query(g, Q, nq, 1, beam, nullptr, idx_out, nullptr, dist_evals);
}

void fmgp_graph_destroy(fmgp_graph* g) {
  if (g == nullptr) return;
  DeviceGuard dg;
  cudaSetDevice(g->device);
  graph_free(g);
}

}  // extern "C"
