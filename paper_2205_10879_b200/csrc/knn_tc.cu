// K1-tc — exact kNN for d >= 4 on the 5th-generation tensor cores:
// a tcgen05 distance GEMM fed by TMA, a per-query threshold filter in the
// TMEM epilogue, and an exact fp64 recheck, so the neighbour indices are the
// reference's bit for bit (proj/core/src/nn_index.cpp:73-81 key,
// :254-287 query_knn, :351-366 nearest).
//
// Data path
//   prep      x^ = fp16(s (x - mu)) row-major, zero-padded to DP = 64*KB columns
//             (one 128-byte swizzle row per 64 dims), mu = mean of the points,
//             s = 2^e the largest power of two with max|x^| <= 2^14 and
//             max_p ||p^||^2 <= 2^16. Three spare columns carry the point norm:
//             points hold the fp16 hi/mid/lo split of -||p^||^2/2, queries hold 1,
//             so the GEMM yields g = q^.p^ - n^_p/2 and v = -2g = D~ - n^_q directly.
//   GEMM      per CTA one 128-query tile (TMEM lanes) x a stream of 128-point
//             tiles (TMEM columns): tcgen05.mma.cta_group::1.kind::f16, M=N=128,
//             K=16, fp32 accumulators in TMEM (4 buffers of 128 columns); TMA
//             (SWIZZLE_128B) feeds a resident query tile + 3 point stages when
//             DP == 64, else 2 stages of (query, point) k-blocks.
//   filter    D~ = n^_q + v approximates s^2 D (D = exact key):
//             |D~ - s^2 D| <= E(D) = 2 eta s sqrt(D) + eta^2 + eps with
//             eta_q = 2^-11 (||q^|| + max||p^||)(1+1e-3) + 2^-24 sqrt(DP) (fp16 input
//             rounding, subnormals included) and eps_q = (2 DP + 32) 2^-22
//             (n^_q + max n^_p)(1+1e-3) + 2^-20 (fp32 accumulation of the dot and
//             norm terms even with truncating adds, the norm split, n^_q in fp32).
//   epilogue  per query an unsorted, append-only candidate buffer (wcap = 64/128/256 (v, index)
//             pairs in a per-CTA global scratch area that stays in L2; an append is one
//             fire-and-forget 8-byte store) holding every point seen so far with
//             v <= win, win = W - n^_q,
//             W = T~ + 2 E(T~), T~ >= the kk-th smallest D~ seen: every point of the
//             exact top-kk is in the buffer at all times. An admission is one
//             shared-memory append; when a query's buffer is full the WARP compacts
//             it (each lane takes cap/32 entries: bisection on the ordered key bits
//             for the kk-th smallest, new window, ballot-prefix compaction), so the
//             expensive step runs on 32 lanes instead of the one diverged lane a
//             per-query heap sift occupies. Per 32-column chunk one max over g
//             decides whether any lane needs it.
//   recheck   tc_recheck_kernel: exact fp64 keys of the buffer from the original
//             coordinates, top-kk by (key, index) — the reference's order. A
//             buffer a compaction cannot shrink flags its query for the fp64 brute force.
// Roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer (one elected
// lane), warps 2-5 epilogue (thread = TMEM lane = query). The epilogue is
// latency-bound with one warp per scheduler, and the candidate state no longer
// lives in shared memory, so TWO CTAs run per SM (256 TMEM columns = 2
// accumulator buffers each, ~85-115 KB of operand stages each): two independent
// query tiles per SM, eight epilogue warps (FMGP_TC_CTAS=1: one CTA per SM
// with deeper operand pipelines).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <climits>
#include <cmath>

#include <cstdio>
#include <cstdlib>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

#ifndef FMGP_TC_RECHECK_CTAS  // CTAs per SM of the grid-stride recheck launch (a few long CTAs per SM leave a tail)
#define FMGP_TC_RECHECK_CTAS 64
#endif
constexpr int kRecheckCtas = FMGP_TC_RECHECK_CTAS;


constexpr int kBM = 128;  // queries per tile (TMEM lanes)
constexpr int kBN = 128;  // reference points per tile (TMEM columns per buffer)
constexpr int kBK = 64;   // fp16 dims per k-block (one 128 B swizzle row)
constexpr int kStages = 2;       // A+B stages when the query tile streams (KB > 1), minimum
constexpr int kStagesMax = 4;    // ... and maximum (as many as shared memory leaves room for)
constexpr int kBStagesRes = 3;   // B-only stages when the query tile is resident (KB == 1), minimum
constexpr int kBStagesResMax = 6;  // ... and maximum
constexpr int kBars = kStagesMax > kBStagesResMax ? kStagesMax : kBStagesResMax;  // stage barriers
constexpr int kTBufs = 2;        // TMEM accumulator buffers per CTA (2 x 128 columns; two CTAs per SM)
constexpr int kCapMax = 128;  // candidates per query handed to the recheck (kk <= kCapMax - 29)
constexpr int kWcapMax = 256;  // working buffer entries per query (8 per lane in a compaction)
constexpr int kMaxThreads = 192;  // TMA + MMA + 4 epilogue warps
constexpr int kScrStride = 36;  // floats per lane scratch row (16 B aligned, spreads banks)
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
constexpr uint32_t kBBytes = kBN * kBK * 2;  // 16 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(su32(bar)),
      "r"(phase)
      : "memory");
}
// Producer-side roles (TMA, MMA) waits. mode 0: spin on try_wait; 1: back off
// with nanosleep; 2: try_wait with a suspend-time hint (the thread sleeps in
// the barrier unit until the phase completes). 1 and 2 keep the roles' spin
// off the issue slots the epilogue warps need (FMGP_TC_WAIT selects, A/B).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase, int mode) {
  if (mode == 2) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONES_%=;\n\t"
        "bra WAITS_%=;\n\t"
        "DONES_%=:\n\t}" ::"r"(su32(bar)),
        "r"(phase), "r"(1000000u)
        : "memory");
    return;
  }
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(su32(bar)), "r"(phase)
        : "memory");
    if (ok) return;
    if (mode == 1) __nanosleep(200);
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// K-major operand in a SWIZZLE_128B tile: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;             // leading byte offset (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024u >> 4) << 32;     // stride byte offset: next 8-row group
  d |= static_cast<uint64_t>(1u) << 46;             // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2u) << 61;             // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: fp16 x fp16 -> fp32, both K-major, M=128, N=kBN.
constexpr uint32_t kIdesc = (1u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(kBN >> 3) << 17) |
                            (static_cast<uint32_t>(kBM >> 4) << 24);

__device__ __forceinline__ void tmem_ld64_nw(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, "
      "%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, "
      "%48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
        "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
        "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
        "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
        "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ prep

__global__ void mean_kernel(const double* __restrict__ P, int64_t np, int d, double* __restrict__ sums) {
  // column sums: thread per (dim, row-chunk)
  for (int t = blockIdx.y * blockDim.x + threadIdx.x; t < d; t += gridDim.y * blockDim.x) {
    double s = 0.0;
    for (int64_t i = blockIdx.x; i < np; i += gridDim.x) s += P[i * d + t];
    atomicAdd(&sums[t], s);
  }
}

__global__ void maxabs_kernel(const double* __restrict__ A, int64_t n, int d, const double* __restrict__ sums,
                              int64_t np, unsigned long long* __restrict__ maxbits) {
  double m = 0.0;
  const int64_t total = n * d;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(e % d);
    m = fmax(m, fabs(A[e] - sums[t] / static_cast<double>(np)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// max_p ||p - mu||^2 (as bits) for the norm-range part of the scale.
__global__ void rownorm_kernel(const double* __restrict__ A, int64_t n, int d, const double* __restrict__ sums,
                               int64_t np, unsigned long long* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  double m = 0.0;
  for (int64_t i = warp; i < n; i += nwarps) {
    double acc = 0.0;
    for (int t = lane; t < d; t += 32) {
      const double v = A[i * d + t] - sums[t] / static_cast<double>(np);
      acc += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    m = fmax(m, acc);
  }
  if (lane == 0) atomicMax(bits, static_cast<unsigned long long>(__double_as_longlong(m)));
}

__device__ __forceinline__ double tc_scale(const unsigned long long* bits) {
  const double maxabs = __longlong_as_double(static_cast<long long>(bits[0]));
  const double maxn2 = __longlong_as_double(static_cast<long long>(bits[2]));
  double s = maxabs > 0.0 ? exp2(floor(log2(16384.0 / maxabs))) : 1.0;
  if (maxn2 > 0.0) s = fmin(s, exp2(floor(0.5 * log2(65536.0 / maxn2))));
  return s;
}

// x^ rows (fp16, DP wide) and n^ = ||x^||^2 (fp32, queries); points also get the
// fp16 split of -n^/2 in columns d..d+2 and max ||x^|| into pmax (as bits),
// queries get 1 in those columns.
__global__ void convert_kernel(const double* __restrict__ A, int64_t n, int d, int DP, const double* __restrict__ sums,
                               int64_t np, const unsigned long long* __restrict__ bits, int is_point,
                               __half* __restrict__ H, float* __restrict__ norms,
                               unsigned long long* __restrict__ pmax_bits) {
  const double s = tc_scale(bits);
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    double acc = 0.0;
    for (int t = lane; t < DP; t += 32) {
      if (t < d) {
        const __half h = __double2half((A[i * d + t] - sums[t] / static_cast<double>(np)) * s);
        const double v = static_cast<double>(__half2float(h));
        acc += v * v;
        H[i * DP + t] = h;
      } else if (t >= d + 3 || !is_point) {
        H[i * DP + t] = __float2half_rn(t < d + 3 ? 1.0f : 0.0f);
      }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (is_point && lane < 3) {  // -acc/2 = c1 + c2 + c3 (+ < 2^-33 relative)
      const double v = -0.5 * acc;
      const __half c1 = __double2half(v);
      const double r1 = v - static_cast<double>(__half2float(c1));
      const __half c2 = __double2half(r1);
      const __half c3 = __double2half(r1 - static_cast<double>(__half2float(c2)));
      H[i * DP + d + lane] = lane == 0 ? c1 : (lane == 1 ? c2 : c3);
    }
    if (lane == 0) {
      if (norms) norms[i] = static_cast<float>(acc);
      if (pmax_bits) atomicMax(pmax_bits, static_cast<unsigned long long>(__double_as_longlong(sqrt(acc))));
    }
  }
}

// ------------------------------------------------------------------ main kernel

struct TcArgs {
  const double* Q;       // nq x d original coordinates (fp64)
  const double* P;       // np x d
  const float* qn;       // ||q^||^2
  int64_t nq, np;
  int d, DP, KB, kk, cap;
  int64_t self_offset;   // exclude p == q + self_offset when >= 0
  const int32_t* excl;   // or per-query exclusion (nullable)
  int with_self;
  int wait_mode;         // producer-side wait (see mbar_wait_sleep)
  int wcap;              // working candidate buffer entries per query (64 / 128 / 256)
  uint2* gbuf;           // [gridDim.x][128][wcap] (v bits, index) working buffers (global scratch, L2)
  int stages;            // pipeline stages: A+B pairs (KB > 1, kStages .. kStagesMax) or B tiles
                         // (KB == 1, kBStagesRes .. kBStagesResMax)
  int nslots;            // 16 KB operand slots: 1 + stages (resident) or 2 * stages
  int32_t* out;          // nq x (kk + with_self)
  double* out_d;         // nq x kk (nullable)
  int32_t* cand;         // [cap][nq] candidate ids, column-major (coalesced stores)
  int32_t* ccount;       // [nq] candidates per query, -1 = overflowed
  int32_t* overflow;     // [0] = count, [1..] = query ids whose list overflowed
  const unsigned long long* maxabs_bits;
  const unsigned long long* pmax_bits;
  float* debug_G;        // when non-null: D~ of (query tile 0, point tile 0) and no search
};

// Admission window W = T + 2 E(T), E(T) = 2 eta (sqrt(T) + 2 eta) + eta^2 + eps (scaled units).
__device__ __forceinline__ float window_of(float T, double eta, double eps) {
  const double t = fmax(static_cast<double>(T), 0.0);  // D~ of a near-duplicate can round below 0
  const double E = 2.0 * eta * (sqrt(t) + 2.0 * eta) + eta * eta + eps;
  return static_cast<float>((t + 2.0 * E) * 1.0001 + 1e-30);
}

// Order-preserving map float -> uint32 (and back) for the selection below.
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t b = __float_as_uint(f);
  return b ^ (static_cast<uint32_t>(static_cast<int32_t>(b) >> 31) | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u ^ 0x80000000u) : ~u);
}

// Warp-cooperative compaction of ONE query's candidate buffer (gb: its n
// (v bits, index) entries, n <= kWcapMax, contiguous in the global scratch
// area; read with ld.global.cg, so the entries other lanes appended or
// compacted are seen from L2). Every lane takes the entries t = lane,
// lane + 32, ...; T = a value with at least kk entries <= T, found by
// bisection on the ordered key bits between the buffer's minimum and maximum
// (exact: T = the kk-th smallest v; otherwise it may stop at the (kk+1)-th);
// the new admission bound is win = W(T + n^_q) - n^_q and the entries above it
// are dropped (ballot-prefix compaction, order preserved). Returns the new
// count; win_out = the new bound. All 32 lanes call it with the same arguments
// (n >= kk).
__device__ __noinline__ int compact_candidates(uint2* gb, int n, int kk, float nqf, double eta, double eps,
                                               bool exact, float* win_out) {
  constexpr int NE = kWcapMax / 32;
  const int lane = threadIdx.x & 31;
  uint2 e[NE];
  uint32_t u[NE];
  uint32_t mn = 0xffffffffu, mx = 0u;
  __syncwarp();
#pragma unroll
  for (int s = 0; s < NE; ++s) {
    const int t = s * 32 + lane;
    const bool in = t < n;
    e[s] = in ? __ldcg(gb + t) : make_uint2(0x7f800000u, 0u);
    u[s] = in ? f2ord(__uint_as_float(e[s].x)) : 0xffffffffu;
    mn = min(mn, u[s]);
    mx = in ? max(mx, u[s]) : mx;
  }
  __syncwarp();
  uint32_t H = __reduce_max_sync(0xffffffffu, mx);      // count(u <= H) = n >= kk
  uint32_t L = __reduce_min_sync(0xffffffffu, mn) - 1u;  // count(u <= L) = 0 < kk
  for (int round = 0; round < 34 && H - L > 1u; ++round) {
    const uint32_t mid = L + ((H - L) >> 1);
    int cl = 0;
#pragma unroll
    for (int s = 0; s < NE; ++s) cl += u[s] <= mid ? 1 : 0;
    const int c = __reduce_add_sync(0xffffffffu, cl);
    if (c >= kk) {
      H = mid;
      if (c == kk || (!exact && c == kk + 1)) break;
    } else {
      L = mid;
    }
  }
  const float win = window_of(ord2f(H) + nqf, eta, eps) - nqf;
  int base = 0;
#pragma unroll
  for (int s = 0; s < NE; ++s) {
    if (s * 32 >= n) break;
    const bool keep = s * 32 + lane < n && __uint_as_float(e[s].x) <= win;
    const uint32_t b = __ballot_sync(0xffffffffu, keep);
    if (keep) gb[base + __popc(b & ((1u << lane) - 1u))] = e[s];
    base += __popc(b);
  }
  __syncwarp();
  *win_out = win;
  return base;
}

__global__ void __launch_bounds__(kMaxThreads, 2)
knn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmP, TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B operands) by offsetting the __shared__ pointer itself,
  // so the compiler keeps the shared address space (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  // 16 KB operand slots: streaming mode (KB > 1) stage s = (A slot s, B slot stages + s);
  // resident mode (KB == 1) A = slot 0 (loaded once per query tile), B stages = slots 1..3
  uint8_t* slots = smem;
  const bool ares = a.KB == 1;
  const int nst = a.stages;
  float* scratch = reinterpret_cast<float*>(slots + a.nslots * kABytes);  // [4 warps][32][kScrStride]
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + 4 * 32 * kScrStride);
  uint64_t* empty = full + kBars;
  uint64_t* tfull = empty + kBars;  // kTBufs TMEM buffers
  uint64_t* tempty = tfull + kTBufs;
  uint64_t* afull = tempty + kTBufs;      // resident query tile
  uint64_t* aempty = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nqt = (a.nq + kBM - 1) / kBM;
  const int64_t npt = (a.np + kBN - 1) / kBN;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kBars; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < kTBufs; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(kTBufs * kBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, aphase = 0;
      for (int64_t qt = blockIdx.x; qt < nqt; qt += gridDim.x) {
        const int64_t pt_end = a.debug_G ? 1 : npt;
        if (ares) {
          mbar_wait_sleep(aempty, aphase ^ 1, a.wait_mode);
          mbar_expect_tx(afull, kABytes);
          tma_load_2d(slots, &tmQ, afull, 0, static_cast<int>(qt * kBM));
          aphase ^= 1;
        }
        for (int64_t pt = 0; pt < pt_end; ++pt) {
          for (int kb = 0; kb < a.KB; ++kb) {
            mbar_wait_sleep(&empty[stage], phase ^ 1, a.wait_mode);
            if (ares) {
              mbar_expect_tx(&full[stage], kBBytes);
              tma_load_2d(slots + (1 + stage) * kABytes, &tmP, &full[stage], 0, static_cast<int>(pt * kBN));
            } else {
              mbar_expect_tx(&full[stage], kStageBytes);
              tma_load_2d(slots + stage * kABytes, &tmQ, &full[stage], kb * kBK, static_cast<int>(qt * kBM));
              tma_load_2d(slots + (nst + stage) * kABytes, &tmP, &full[stage], kb * kBK, static_cast<int>(pt * kBN));
            }
            if (++stage == nst) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    int stage = 0;
    uint32_t phase = 0, aphase = 0;
    int buf = 0;
    uint32_t tphase = 0;
    for (int64_t qt = blockIdx.x; qt < nqt; qt += gridDim.x) {
      const int64_t pt_end = a.debug_G ? 1 : npt;
      if (ares) {
        mbar_wait(afull, aphase);
        aphase ^= 1;
      }
      for (int64_t pt = 0; pt < pt_end; ++pt) {
        mbar_wait_sleep(&tempty[buf], tphase ^ 1, a.wait_mode);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(buf * kBN);
        for (int kb = 0; kb < a.KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint64_t ad = sdesc_sw128(su32(ares ? slots : slots + stage * kABytes));
            const uint64_t bd = sdesc_sw128(su32(slots + (ares ? 1 + stage : nst + stage) * kABytes));
#pragma unroll
            for (int k16 = 0; k16 < kBK / 16; ++k16)
              tc_mma_f16(d_tmem, ad + 2 * k16, bd + 2 * k16, kIdesc, (kb > 0 || k16 > 0) ? 1u : 0u);
            tc_commit(&empty[stage]);
            if (kb == a.KB - 1) tc_commit(&tfull[buf]);
          }
          __syncwarp();
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (++buf == kTBufs) {
          buf = 0;
          tphase ^= 1;
        }
      }
      if (ares) {
        if (lane == 0) tc_commit(aempty);  // query tile free once this tile's MMAs complete
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue: thread = TMEM lane = query row of the tile
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int ew = warp - 2;       // epilogue warp 0 .. 3
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    const double pmax = __longlong_as_double(static_cast<long long>(*a.pmax_bits));
    float* scr = scratch + (ew * 32 + lane) * kScrStride;  // this lane's hot-chunk values
    // this warp's 32 candidate buffers in the CTA's global scratch area (lane l: + l * wcap)
    uint2* wb0 = a.gbuf + (static_cast<int64_t>(blockIdx.x) * kBM + quarter * 32) * a.wcap;
    uint2* gb = wb0 + lane * a.wcap;  // this query's buffer
    int buf = 0;
    uint32_t tphase = 0;
    for (int64_t qt = blockIdx.x; qt < nqt; qt += gridDim.x) {
      const int64_t q = qt * kBM + row;
      const bool valid = q < a.nq;
      const double nq_hat = valid ? static_cast<double>(a.qn[q]) : 0.0;
      const float nqf = static_cast<float>(nq_hat);
      const double eta = 4.8828125e-4 * (sqrt(nq_hat) + pmax) * 1.001 + 5.9604644775390625e-8 * sqrt(double(a.DP));
      const double eps = (2 * a.DP + 32) * 2.384185791015625e-7 * (nq_hat + pmax * pmax) * 1.001 + 9.5367431640625e-7;
      const int64_t excl = a.excl != nullptr ? (valid ? a.excl[q] : -1)
                                             : (a.self_offset >= 0 ? q + a.self_offset : -1);
      // Candidate state: gb[0..cnt) = every point seen so far with v <= win (unsorted).
      // win = +inf until the first compaction (cnt reaches wcap >= kk + 29), then
      // W(T~) - n^_q with T~ >= the kk-th smallest D~ seen, so the exact top-kk is inside.
      int cnt = 0;
      bool over = false;
      float win = valid ? INFINITY : -INFINITY;  // admission bound on D~ - n^_q
      const int64_t pt_end = a.debug_G ? 1 : npt;
      for (int64_t pt = 0; pt < pt_end; ++pt) {
        mbar_wait(&tfull[buf], tphase);
        tc_fence_after();
        const uint32_t tbase = tmem_base + lane_addr + static_cast<uint32_t>(buf * kBN);
        const bool tail = (pt + 1) * kBN > a.np;  // columns past np hold TMA zero fill
        // 64 columns per step (tcgen05.ld x64): the filter of a step is one dependent chain
        // (load -> eight 8-column maxima -> eight votes -> branch) and the epilogue warp has
        // at most one other warp on its scheduler to hide it, so fewer, wider steps.
        // Admissions of one 32-column half: per-lane bit mask of the hot sub-chunks, their
        // v = -2g parked in this lane's scratch row, so the append loop visits only set bits;
        // a lane whose buffer is full stops with its remaining bits pending, the warp
        // compacts those lanes' buffers one by one, and the lanes go on.
        auto admit_half = [&](uint32_t (&r)[64], const int off, const uint32_t hot4, const int64_t j0,
                              const float gthr) {
          uint32_t mask = 0;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            if (((hot4 >> q4) & 1u) == 0) continue;
            const int c = 8 * q4, o = off + c;
#pragma unroll
            for (int t = 0; t < 8; ++t) mask |= (__uint_as_float(r[o + t]) >= gthr ? 1u : 0u) << (c + t);
            *reinterpret_cast<float4*>(scr + c) =
                make_float4(-2.0f * __uint_as_float(r[o]), -2.0f * __uint_as_float(r[o + 1]),
                            -2.0f * __uint_as_float(r[o + 2]), -2.0f * __uint_as_float(r[o + 3]));
            *reinterpret_cast<float4*>(scr + c + 4) =
                make_float4(-2.0f * __uint_as_float(r[o + 4]), -2.0f * __uint_as_float(r[o + 5]),
                            -2.0f * __uint_as_float(r[o + 6]), -2.0f * __uint_as_float(r[o + 7]));
          }
          for (;;) {
            while (mask != 0 && cnt < a.wcap) {
              const int c = __ffs(mask) - 1;
              mask &= mask - 1;
              const float v = scr[c];
              const int64_t j = j0 + c;
              if (!(v <= win) || j == excl) continue;
              gb[cnt] = make_uint2(__float_as_uint(v), static_cast<uint32_t>(j));
              ++cnt;
            }
            uint32_t need = __ballot_sync(0xffffffffu, mask != 0);
            if (need == 0) break;
            while (need != 0) {
              const int src = __ffs(need) - 1;
              need &= need - 1;
              const float s_nqf = __shfl_sync(0xffffffffu, nqf, src);
              const double s_eta = __shfl_sync(0xffffffffu, eta, src);
              const double s_eps = __shfl_sync(0xffffffffu, eps, src);
              float nwin;
              const int nn = compact_candidates(wb0 + src * a.wcap, a.wcap, a.kk, s_nqf, s_eta, s_eps, false, &nwin);
              if (lane == src) {
                cnt = nn;
                win = nwin;
                if (nn > a.wcap - 32) {  // the window alone (nearly) fills the buffer: the query is redone exactly
                  over = true;
                  win = -INFINITY;
                  mask = 0;
                  cnt = 0;
                }
              }
            }
          }
        };
#pragma unroll 1
        for (int h = 0; h < kBN / 64; ++h) {
          uint32_t r[64];
          __syncwarp();  // tcgen05.ld is warp-collective; the admission loop diverges
          tmem_ld64_nw(tbase + h * 64, r);
          tmem_wait_ld();
          const int64_t j0 = pt * kBN + h * 64;
          if (tail) {  // NaN: never admitted, ignored by the max
#pragma unroll
            for (int c = 0; c < 64; ++c)
              if (j0 + c >= a.np) r[c] = 0x7fffffffu;
          }
          if (a.debug_G) {
            if (qt == 0)
              for (int c = 0; c < 64; ++c)
                a.debug_G[row * 256 + h * 64 + c] = j0 + c < a.np ? fmaf(-2.0f, __uint_as_float(r[c]), nqf) : 0.0f;
            continue;
          }
          // g_c = q^.p^ - n^_p/2 straight from TMEM; an 8-column sub-chunk whose max g is
          // below -win/2 (for every lane) has nothing under the window
          const float gthr = -0.5f * win;  // v <= win  <=>  g >= -win/2 (exact scaling)
          uint32_t hot = 0;
#pragma unroll
          for (int q8 = 0; q8 < 8; ++q8) {
            const int c = 8 * q8;
            const float m8 = fmaxf(fmaxf(fmaxf(__uint_as_float(r[c]), __uint_as_float(r[c + 1])),
                                         fmaxf(__uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]))),
                                   fmaxf(fmaxf(__uint_as_float(r[c + 4]), __uint_as_float(r[c + 5])),
                                         fmaxf(__uint_as_float(r[c + 6]), __uint_as_float(r[c + 7]))));
            hot |= (__any_sync(0xffffffffu, m8 >= gthr) ? 1u : 0u) << q8;
          }
          if (hot == 0) continue;
          if ((hot & 15u) != 0) admit_half(r, 0, hot & 15u, j0, gthr);
          // the second half sees the bound the first half's compactions may have tightened
          // through `win` only at the append (v <= win); gthr stays the looser, still valid bound
          if ((hot >> 4) != 0) admit_half(r, 32, hot >> 4, j0 + 32, gthr);
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);
        if (++buf == kTBufs) {
          buf = 0;
          tphase ^= 1;
        }
      }
      // candidates = the buffer (the exact top-kk is inside), trimmed once more to the final
      // window (exact kk-th smallest); the exact recheck and selection run in tc_recheck_kernel
      if (a.debug_G) continue;
      {
        uint32_t need = __ballot_sync(0xffffffffu, valid && !over && cnt > a.kk);
        while (need != 0) {
          const int src = __ffs(need) - 1;
          need &= need - 1;
          const float s_nqf = __shfl_sync(0xffffffffu, nqf, src);
          const double s_eta = __shfl_sync(0xffffffffu, eta, src);
          const double s_eps = __shfl_sync(0xffffffffu, eps, src);
          const int s_cnt = __shfl_sync(0xffffffffu, cnt, src);
          float nwin;
          const int nn = compact_candidates(wb0 + src * a.wcap, s_cnt, a.kk, s_nqf, s_eta, s_eps, true, &nwin);
          if (lane == src) cnt = nn;
        }
      }
      __syncwarp();
      if (!valid) continue;
      if (cnt > a.cap) over = true;  // more candidates inside the final window than the recheck takes
      if (over) {
        const int32_t slot = atomicAdd(a.overflow, 1);
        a.overflow[1 + slot] = static_cast<int32_t>(q);
        a.ccount[q] = -1;
        continue;
      }
      int32_t* cq = a.cand + q;
      for (int t = 0; t < cnt; ++t) cq[t * a.nq] = static_cast<int32_t>(__ldcg(gb + t).y);
      a.ccount[q] = cnt;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTBufs * kBN));
  }
}

// Exact recheck, one warp per query: fp64 keys of the (<= cap <= 128)
// candidates with the reference's sequential difference order, then each
// candidate's rank under (key, index) by broadcasting all candidates through
// the warp; rank < kk goes straight to its output slot.
constexpr int kRecheckWarps = 4;

__global__ void __launch_bounds__(kRecheckWarps * 32) tc_recheck_kernel(const double* __restrict__ Q, const double* __restrict__ P,
                                                          int d, int64_t nq, int kk, const int32_t* __restrict__ cand,
                                                          const int32_t* __restrict__ ccount, int halves, int cap,
                                                          int with_self,
                                                          int64_t self_offset, int32_t* __restrict__ out,
                                                          double* __restrict__ out_d) {
  __shared__ double rtile[kRecheckWarps * (32 * 33 + 32)];
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = w0; q < nq; q += nw) {
    const int cnt0 = ccount[q];
    const int cnt1 = halves == 2 ? ccount[nq + q] : 0;
    if (cnt0 < 0 || cnt1 < 0) continue;  // overflowed: redone by the brute-force path
    const int cnt = cnt0 + cnt1;          // <= 128 (host: halves == 2 only when 2 cap <= 128)
    const double* qx = Q + q * d;
    double key[4];
    int32_t idx[4];
    int rank[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int t = s * 32 + lane;
      rank[s] = 0;
      if (t < cnt) {
        const int row_c = t < cnt0 ? t : cap + (t - cnt0);  // half 1's candidates start at row cap
        idx[s] = cand[static_cast<int64_t>(row_c) * nq + q];
      } else {
        idx[s] = INT_MAX;
      }
      key[s] = INFINITY;
    }
    if (d < 16) {
#pragma unroll
      for (int s = 0; s < 4; ++s)
        if (idx[s] != INT_MAX) key[s] = dist_sq_dyn(qx, P + static_cast<int64_t>(idx[s]) * d, d);
    } else {
      // wide rows: 32 candidate rows x 32 dims staged through this warp's padded
      // tile with coalesced loads; each lane then accumulates its own candidate's
      // key over the dims in ascending order (the reference's bit-exact key)
      double* tl = rtile + (threadIdx.x >> 5) * (32 * 33 + 32);
      double* qt = tl + 32 * 33;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (s * 32 >= cnt) break;
        double acc = 0.0;
        for (int c0 = 0; c0 < d; c0 += 32) {
          const int dc = min(32, d - c0);
          __syncwarp();
          qt[lane] = lane < dc ? qx[c0 + lane] : 0.0;
          for (int r = 0; r < 32; ++r) {
            const int32_t ir = __shfl_sync(0xffffffffu, idx[s], r);
            if (ir != INT_MAX && lane < dc) tl[r * 33 + lane] = P[static_cast<int64_t>(ir) * d + c0 + lane];
          }
          __syncwarp();
          for (int c = 0; c < dc; ++c) {
            const double e = __dsub_rn(qt[c], tl[lane * 33 + c]);
            acc = __dadd_rn(acc, __dmul_rn(e, e));
          }
        }
        if (idx[s] != INT_MAX) key[s] = acc;
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
      if (s2 * 32 >= cnt) break;
      for (int l = 0; l < 32; ++l) {
        const double ku = __shfl_sync(0xffffffffu, key[s2], l);
        const int32_t iu = __shfl_sync(0xffffffffu, idx[s2], l);
#pragma unroll
        for (int s = 0; s < 4; ++s) rank[s] += pair_less(ku, iu, key[s], idx[s]) ? 1 : 0;
      }
    }
    const int width = kk + (with_self ? 1 : 0);
    int32_t* orow = out + q * width + (with_self ? 1 : 0);
    if (with_self && lane == 0) out[q * width] = static_cast<int32_t>(q + self_offset);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (s * 32 + lane < cnt && rank[s] < kk) {
        orow[rank[s]] = idx[s];
        if (out_d) out_d[q * kk + rank[s]] = key[s];
      }
    }
    for (int t = cnt + lane; t < kk; t += 32) {  // fewer candidates than kk (np < kk)
      orow[t] = INT_MAX;
      if (out_d) out_d[q * kk + t] = INFINITY;
    }
  }
}

// Redo the overflowed queries exactly (brute force): gather their rows, run
// the fp64 scan with per-query exclusion, scatter the rows back.
__global__ void gather_rows_kernel(const double* __restrict__ Q, int d, const int32_t* __restrict__ ids, int cnt,
                                   int64_t self_offset, const int32_t* __restrict__ excl_in, double* __restrict__ Qg,
                                   int32_t* __restrict__ excl_out) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < static_cast<int64_t>(cnt) * d;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / d), t = static_cast<int>(e % d);
    const int64_t q = ids[r];
    Qg[e] = Q[q * d + t];
    if (t == 0)
      excl_out[r] = excl_in != nullptr ? excl_in[q] : (self_offset >= 0 ? static_cast<int32_t>(q + self_offset) : -1);
  }
}

__global__ void scatter_rows_kernel(const int32_t* __restrict__ rows, const double* __restrict__ rows_d,
                                    const int32_t* __restrict__ ids, int cnt, int kk, int with_self,
                                    int64_t self_offset, int32_t* __restrict__ out, double* __restrict__ out_d) {
  const int width = kk + (with_self ? 1 : 0);
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < static_cast<int64_t>(cnt) * kk;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / kk), t = static_cast<int>(e % kk);
    const int64_t q = ids[r];
    if (with_self && t == 0) out[q * width] = static_cast<int32_t>(q + self_offset);
    out[q * width + (with_self ? 1 : 0) + t] = rows[e];
    if (out_d) out_d[q * kk + t] = rows_d[e];
  }
}

bool make_map(CUtensorMap* map, const __half* ptr, int64_t rows, int DP, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (encode == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || fn == nullptr)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(DP), static_cast<cuuint64_t>(rows)};
  cuuint64_t gstride[1] = {static_cast<cuuint64_t>(DP) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(ptr), gdim, gstride, box, estride,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

unsigned g1(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<unsigned>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

bool knn_tc_supported(int d, int kk) { return d >= 4 && d <= 1024 && kk >= 1 && kk <= kCapMax - 29; }

cudaError_t knn_tc(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk, int64_t self_offset,
                   const int32_t* excl_arr, int with_self, int32_t* out, double* out_d, int num_sms,
                   cudaStream_t s, float* debug_G) {
  if (nq <= 0) return cudaSuccess;
  const int KB = (d + 3 + kBK - 1) / kBK;  // + 3 columns for the point-norm split
  const int DP = KB * kBK;
  const int cap = kCapMax;  // candidates per query the recheck takes (rows of `cand`)
  // working buffer per query: the first wcap points are all admitted, then every compaction
  // leaves >= kk entries, so the slack wcap - kk sets how often a query compacts
  const int wcap = kk > 64 ? kWcapMax : (kk > 16 ? 128 : 64);
  // Two CTAs per SM (the epilogue is latency-bound with one warp per scheduler); each gets
  // half of the SM's shared memory for its operand stages. FMGP_TC_CTAS=1: one CTA per SM.
  // With no more query tiles than SMs a second CTA per SM has nothing to run: one CTA, deep stages.
  const char* cta_env = std::getenv("FMGP_TC_CTAS");
  const int ctas = (cta_env != nullptr && cta_env[0] == '1') || (nq + kBM - 1) / kBM <= num_sms ? 1 : 2;
  const size_t smem_cap = ctas == 2 ? (233472 - 2 * 1024) / 2 : 232448;
  auto smem_for = [&](int nslots) {
    return static_cast<size_t>(1024) + static_cast<size_t>(nslots) * kABytes + sizeof(float) * 4 * 32 * kScrStride + 256;
  };
  // As many operand stages in flight as fit (the TMA round trip from L2 is several MMA
  // k-blocks long): (A, B) k-block pairs for wide rows, B tiles when the query tile is
  // resident. FMGP_TC_STAGES overrides (A/B checks).
  const char* st_env = std::getenv("FMGP_TC_STAGES");
  const int smin = KB > 1 ? kStages : kBStagesRes, smax = KB > 1 ? kStagesMax : kBStagesResMax;
  const int want = st_env != nullptr ? std::atoi(st_env) : smax;
  int stages = smin;
  for (int st = std::min(std::max(want, smin), smax); st >= smin; --st)
    if (smem_for(KB > 1 ? 2 * st : 1 + st) <= smem_cap) {
      stages = st;
      break;
    }
  const int nslots = KB > 1 ? 2 * stages : 1 + stages;
  __half *Qh = nullptr, *Ph = nullptr;
  float* qn = nullptr;
  double* sums = nullptr;
  int32_t *cand = nullptr, *ccount = nullptr, *ovf = nullptr;
  uint2* gbuf = nullptr;
  const int64_t nqt = (nq + kBM - 1) / kBM;
  const int grid = debug_G ? 1 : static_cast<int>(std::min<int64_t>(nqt, static_cast<int64_t>(num_sms) * ctas));
  unsigned long long* bits = nullptr;  // [0] maxabs, [1] pmax, [2] max ||p - mu||^2
  cudaError_t err = cudaMallocAsync(&Qh, sizeof(__half) * nq * DP, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&Ph, sizeof(__half) * np * DP, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&qn, sizeof(float) * nq, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&sums, sizeof(double) * d, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&bits, sizeof(unsigned long long) * 3, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&cand, sizeof(int32_t) * nq * cap, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&ccount, sizeof(int32_t) * nq, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&gbuf, sizeof(uint2) * static_cast<size_t>(grid) * kBM * wcap, s);
  if (err == cudaSuccess) err = cudaMallocAsync(&ovf, sizeof(int32_t) * (nq + 1), s);
  if (err != cudaSuccess) return err;
  cudaMemsetAsync(sums, 0, sizeof(double) * d, s);
  cudaMemsetAsync(bits, 0, sizeof(unsigned long long) * 3, s);
  cudaMemsetAsync(ovf, 0, sizeof(int32_t), s);
  mean_kernel<<<dim3(256, (d + 255) / 256), 256, 0, s>>>(P, np, d, sums);
  maxabs_kernel<<<g1(np * d), 256, 0, s>>>(P, np, d, sums, np, bits);
  if (Q != P) maxabs_kernel<<<g1(nq * d), 256, 0, s>>>(Q, nq, d, sums, np, bits);
  rownorm_kernel<<<g1(np * 32), 256, 0, s>>>(P, np, d, sums, np, bits + 2);
  convert_kernel<<<g1(np * 32), 256, 0, s>>>(P, np, d, DP, sums, np, bits, 1, Ph, nullptr, bits + 1);
  convert_kernel<<<g1(nq * 32), 256, 0, s>>>(Q, nq, d, DP, sums, np, bits, 0, Qh, qn, nullptr);
  note_launches(Q != P ? 6 : 5);

  CUtensorMap mq, mp;
  if (!make_map(&mq, Qh, nq, DP, kBM) || !make_map(&mp, Ph, np, DP, kBN)) return cudaErrorInvalidValue;
  TcArgs a;
  a.Q = Q;
  a.P = P;
  a.qn = qn;
  a.nq = nq;
  a.np = np;
  a.d = d;
  a.DP = DP;
  a.KB = KB;
  a.kk = kk;
  a.cap = cap;
  a.wcap = wcap;
  a.gbuf = gbuf;
  a.stages = stages;
  a.nslots = nslots;
  a.self_offset = self_offset;
  a.excl = excl_arr;
  a.with_self = with_self;
  {
    static const int wm = [] {
      const char* e = std::getenv("FMGP_TC_WAIT");
      if (e == nullptr) return 1;
      return e[0] == 's' && e[1] == 'p' ? 0 : (e[0] == 'h' ? 2 : 1);
    }();
    a.wait_mode = wm;
  }
  a.out = out;
  a.out_d = out_d;
  a.cand = cand;
  a.ccount = ccount;
  a.overflow = ovf;
  a.maxabs_bits = bits;
  a.pmax_bits = bits + 1;
  a.debug_G = debug_G;
  const size_t smem = smem_for(nslots);
  err = cudaFuncSetAttribute(knn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  knn_tc_kernel<<<grid, kMaxThreads, smem, s>>>(mq, mp, a);
  note_launches(1);
  err = cudaGetLastError();
  if (err == cudaSuccess && debug_G == nullptr) {
    const int64_t blocks = (nq + kRecheckWarps - 1) / kRecheckWarps;
    tc_recheck_kernel<<<static_cast<unsigned>(blocks < num_sms * kRecheckCtas ? blocks : num_sms * kRecheckCtas), kRecheckWarps * 32, 0,
                        s>>>(
        Q, P, d, nq, kk, cand, ccount, 1, cap, with_self, self_offset, out, out_d);
    note_launches(1);
    err = cudaGetLastError();
  }
  if (err == cudaSuccess && debug_G == nullptr) {
    // exact fallback for the (rare) queries whose candidate window overflowed
    int32_t novf = 0;
    err = cudaMemcpyAsync(&novf, ovf, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (err == cudaSuccess) err = cudaStreamSynchronize(s);
    if (err == cudaSuccess && std::getenv("FMGP_TC_STATS") != nullptr)
      std::fprintf(stderr, "knn_tc: nq=%lld np=%lld kk=%d wcap=%d ctas/SM=%d stages=%d overflowed=%d\n",
                   static_cast<long long>(nq), static_cast<long long>(np), kk, wcap, ctas, stages, novf);
    if (err == cudaSuccess && novf > 0) {
      double *Qg = nullptr, *rd = nullptr;
      int32_t *eg = nullptr, *rows = nullptr;
      err = cudaMallocAsync(&Qg, sizeof(double) * novf * d, s);
      if (err == cudaSuccess) err = cudaMallocAsync(&eg, sizeof(int32_t) * novf, s);
      if (err == cudaSuccess) err = cudaMallocAsync(&rows, sizeof(int32_t) * novf * kk, s);
      if (err == cudaSuccess) err = cudaMallocAsync(&rd, sizeof(double) * novf * kk, s);
      if (err == cudaSuccess) {
        gather_rows_kernel<<<g1(static_cast<int64_t>(novf) * d), 256, 0, s>>>(Q, d, ovf + 1, novf, self_offset,
                                                                              excl_arr, Qg, eg);
        err = knn_bruteforce(Qg, novf, P, np, d, kk, -1, eg, 0, rows, rd, num_sms, s);
        scatter_rows_kernel<<<g1(static_cast<int64_t>(novf) * kk), 256, 0, s>>>(rows, rd, ovf + 1, novf, kk,
                                                                                with_self, self_offset, out, out_d);
        note_launches(2);
      }
      for (void* p : {static_cast<void*>(Qg), static_cast<void*>(eg), static_cast<void*>(rows), static_cast<void*>(rd)})
        if (p) cudaFreeAsync(p, s);
    }
  }
  for (void* p : {static_cast<void*>(Qh), static_cast<void*>(Ph), static_cast<void*>(qn),
                  static_cast<void*>(sums), static_cast<void*>(bits), static_cast<void*>(cand), static_cast<void*>(ccount),
                  static_cast<void*>(ovf), static_cast<void*>(gbuf)})
    cudaFreeAsync(p, s);
  return err;
}

}  // namespace fmgp
