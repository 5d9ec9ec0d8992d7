// FP64 pipe peak on this B200 (MEASURED_PEAKS.json has only HBM and bf16).
// Measures the issue rate of independent DADD/DMUL (the non-FMA ops the exact
// kNN key and the kernel build use) and of DFMA, over the whole chip, with
// CUDA events. Prints one JSON object.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void addmul(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      x[c] = __dadd_rn(x[c], a);
      x[c] = __dmul_rn(x[c], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void fmaop(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

// DMMA (mma.sync.m8n8k4.f64) issue rate: 8 independent accumulator chains.
__global__ void dmmaop(double* out, double a, double b) {
  double c[kChains][2];
#pragma unroll
  for (int q = 0; q < kChains; ++q) c[q][0] = c[q][1] = threadIdx.x * 1e-3 + q;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(c[q][0]), "+d"(c[q][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

// Mixed: each warp interleaves one DMMA chain step with 8 DFMA chains per
// iteration (the same per-warp DMMA and DFMA work as half of each kernel
// above): time ~ max(parts) if DMMA and DFMA use separate units, ~ sum if shared.
__global__ void mixedop(double* out, double a, double b) {
  double x[kChains];
  double c[kChains / 2][2];
#pragma unroll
  for (int q = 0; q < kChains; ++q) x[q] = threadIdx.x * 1e-3 + q;
#pragma unroll
  for (int q = 0; q < kChains / 2; ++q) c[q][0] = c[q][1] = threadIdx.x * 1e-3 + q;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int q = 0; q < kChains / 2; ++q)
      asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(c[q][0]), "+d"(c[q][1])
          : "d"(a), "d"(b));
#pragma unroll
    for (int q = 0; q < kChains; ++q) {
      x[q] = fma(x[q], a, b);
      if (q & 1) x[q] = fma(x[q], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kChains; ++q) s += x[q];
#pragma unroll
  for (int q = 0; q < kChains / 2; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  dim3 grid(sms * 8), block(256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best_am = 1e30f, best_f = 1e30f, best_mma = 1e30f, best_mix = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0);
    addmul<<<grid, block>>>(out, 1e-9, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best_am) best_am = ms;
    cudaEventRecord(e0);
    fmaop<<<grid, block>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best_f) best_f = ms;
    cudaEventRecord(e0);
    dmmaop<<<grid, block>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best_mma) best_mma = ms;
    cudaEventRecord(e0);
    mixedop<<<grid, block>>>(out, 0.999999, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best_mix) best_mix = ms;
  }
  double threads = double(grid.x) * block.x;
  double ops_am = threads * kIters * kChains * 2;  // DADD + DMUL
  double ops_f = threads * kIters * kChains;       // DFMA
  double tops_am = ops_am / (best_am * 1e-3) / 1e12;
  double tflops_f = 2 * ops_f / (best_f * 1e-3) / 1e12;
  double warps = threads / 32;
  double tflops_mma = warps * kIters * kChains * 512.0 / (best_mma * 1e-3) / 1e12;  // 8x8x4 FMAs = 512 flops
  printf("{\"fp64_tops_nonfma\": %.3f, \"fp64_dfma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"sms\": %d, \"clock_khz_attr\": %d, "
         "\"ops_per_clk_per_sm_nonfma_at_attr_clock\": %.2f, \"how\": \"independent DADD+DMUL chains (1 op each) and "
         "DFMA chains (2 flops), DMMA m8n8k4 chains (512 flops), %d blocks x 256 threads x %d chains x %d iters, best of 5, CUDA events\"}\n",
         tops_am, tflops_f, tflops_mma, sms, clk, tops_am * 1e12 / (sms * (clk * 1e3)), grid.x, kChains, kIters);
  // mixed: 4 DMMA chains (half the dmma kernel's MMAs) + 12 DFMA per iter (1.5x half the fma kernel's)
  double t_dmma_part = best_mma * 0.5, t_dfma_part = best_f * 12.0 / 8.0;
  printf("{\"mixed_ms\": %.3f, \"dmma_part_ms\": %.3f, \"dfma_part_ms\": %.3f, \"sum_ms\": %.3f, \"max_ms\": %.3f, "
         "\"how\": \"per warp per iter: 4 DMMA m8n8k4 + 12 DFMA; separate units if mixed ~ max, shared if ~ sum\"}\n",
         best_mix, t_dmma_part, t_dfma_part, t_dmma_part + t_dfma_part,
         t_dmma_part > t_dfma_part ? t_dmma_part : t_dfma_part);
  return 0;
}
