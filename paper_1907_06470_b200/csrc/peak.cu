// FP64 peak microbenchmarks: the roofline denominator for the f64 tile GEMM.
//
// MEASURED_PEAKS.json (driver-written) carries HBM and bf16 peaks only; FP64
// has no tcgen05 kind on sm_100a, so the relevant tensor peak is the legacy
// DMMA pipe (mma.sync.m8n8k4.f64). These kernels saturate it (and, for
// comparison, the DFMA pipe) with independent accumulator chains on every SM
// and report FLOP/s from CUDA events.
#include <algorithm>

#include "common.cuh"

namespace xb {
namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dmma_peak_kernel(int iters, double* sink) {
  double d[kChains][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1])
                   : "d"(a), "d"(b));
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += d[c][0] + d[c][1];
  if (acc == 12345.678) sink[0] = acc;
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(int iters, double* sink) {
  double d[kChains];
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
#pragma unroll
  for (int c = 0; c < kChains; ++c) d[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c] = fma(d[c], a, b);
  }
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += d[c];
  if (acc == 12345.678) sink[0] = acc;
}

}  // namespace

// Returns TFLOP/s for the DMMA and DFMA pipes (best of `reps`).
void measure_fp64_peaks(cudaStream_t st, double* dmma_tflops, double* dfma_tflops) {
  double* sink = nullptr;
  XB_CUDA(cudaMalloc(&sink, sizeof(double)));
  cudaEvent_t e0, e1;
  XB_CUDA(cudaEventCreate(&e0));
  XB_CUDA(cudaEventCreate(&e1));
  const int blocks = kNumSMs * 4, threads = 256, iters = 4096;
  auto run = [&](bool mma) {
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
      XB_CUDA(cudaEventRecord(e0, st));
      if (mma)
        dmma_peak_kernel<<<blocks, threads, 0, st>>>(iters, sink);
      else
        dfma_peak_kernel<<<blocks, threads, 0, st>>>(iters, sink);
      check_launch("fp64_peak");
      XB_CUDA(cudaEventRecord(e1, st));
      XB_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      XB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      const double warps = (double)blocks * threads / 32.0;
      const double flops = mma ? warps * iters * kChains * 512.0  // 8x8x4 x 2 per warp-op
                               : (double)blocks * threads * iters * kChains * 2.0;
      best = std::max(best, flops / (ms * 1e-3) / 1e12);
    }
    return best;
  };
  *dmma_tflops = run(true);
  *dfma_tflops = run(false);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
}

}  // namespace xb
