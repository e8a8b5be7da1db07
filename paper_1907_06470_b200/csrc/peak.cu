// FP64 peak microbenchmarks: the roofline denominator for the f64 tile GEMM.
//
// MEASURED_PEAKS.json (driver-written) carries HBM and bf16 peaks only; FP64
// has no tcgen05 kind on sm_100a, so the relevant tensor peak is the legacy
// DMMA pipe (mma.sync.m8n8k4.f64). These kernels saturate it (and, for
// comparison, the DFMA pipe) with independent accumulator chains on every SM
// and report FLOP/s from CUDA events.
#include <algorithm>

#include "common.cuh"
#include "tc_util.cuh"

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

// ---- tcgen05 tensor-pipe peaks: kind::i8 (the Ozaki GEMMs' pipe) and
// kind::f16 with bf16 inputs (to check the method against MEASURED_PEAKS.json)
//
// One CTA per SM; one elected thread issues back-to-back
// tcgen05.mma.cta_group::1 (M=128, N=256, K=32 bytes of each operand) from
// two fixed shared-memory tiles (no-swizzle K-major, the layout ozgemm reads)
// into two alternating TMEM accumulators (2 x 256 columns), with a commit
// every 32 MMAs so the issue queue never drains. No loads: the tensor pipe
// alone bounds it. Ops = 2 M N K per MMA (K = 32 int8 or 16 bf16).
namespace {

template <bool I8>
__global__ void __launch_bounds__(128) tc_peak_kernel(int iters, int random_data) {
  __shared__ __align__(1024) uint8_t a_s[128 * 32];
  __shared__ __align__(1024) uint8_t b_s[256 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  // operand bytes: small constants, or (random_data) uniformly random bytes —
  // the digit slices of real data toggle every input bit of the tensor core,
  // and its power draw, hence the SM clock it sustains, depends on that
  auto mix = [](uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
  };
  for (int i = threadIdx.x; i < 128 * 32 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(a_s)[i] =
        random_data ? (I8 ? mix(i + 977u * blockIdx.x) : (mix(i) & 0x3fff3fffu) | 0x30003000u)
                    : 0x01010101u * (i & 3);
  for (int i = threadIdx.x; i < 256 * 32 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(b_s)[i] =
        random_data ? (I8 ? mix(i + 7919u + 31u * blockIdx.x) : (mix(i + 99u) & 0x3fff3fffu) | 0x30003000u)
                    : 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        tc::su32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x == 0) {
    // D s32 (2) / f32 (1); A, B signed int8 (1) / bf16 (1); N = 256, M = 128
    const uint32_t idesc = (I8 ? (2u << 4) : (1u << 4)) | (1u << 7) | (1u << 10) |
                           ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t da = tc::smem_desc(tc::su32(a_s), 256, 0, 128);
    const uint64_t db = tc::smem_desc(tc::su32(b_s), 256, 0, 128);
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const uint32_t d = tmem + (uint32_t)((j & 1) * 256);
        if (I8)
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(da), "l"(db), "r"(idesc), "r"(it | (j >> 1)));
        else
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(da), "l"(db), "r"(idesc), "r"(it | (j >> 1)));
      }
      // keep at most ~2 batches in flight
      tc::mma_commit(&bar);
      if (it > 0) {
        tc::mbar_wait(&bar, phase);
        phase ^= 1;
      }
    }
    tc::mbar_wait(&bar, phase);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

}  // namespace

// Dense tensor-pipe rates of this device (best of 4): int8 TOP/s
// (tcgen05.mma kind::i8) and bf16 TFLOP/s (kind::f16, f32 accumulate).
void measure_tc_peaks(cudaStream_t st, double* i8_tops, double* bf16_tflops, int random_data) {
  cudaEvent_t e0, e1;
  XB_CUDA(cudaEventCreate(&e0));
  XB_CUDA(cudaEventCreate(&e1));
  const int blocks = kNumSMs, iters = 2048;
  auto run = [&](bool i8) {
    double best = 0.0;
    for (int rep = 0; rep < 4; ++rep) {
      XB_CUDA(cudaEventRecord(e0, st));
      if (i8)
        tc_peak_kernel<true><<<blocks, 128, 0, st>>>(iters, random_data);
      else
        tc_peak_kernel<false><<<blocks, 128, 0, st>>>(iters, random_data);
      check_launch("tc_peak");
      XB_CUDA(cudaEventRecord(e1, st));
      XB_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      XB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      const double ops = (double)blocks * iters * 32 * 2.0 * 128 * 256 * (i8 ? 32 : 16);
      best = std::max(best, ops / (ms * 1e-3) / 1e12);
    }
    return best;
  };
  run(true);  // warm the clocks
  *i8_tops = run(true);
  *bf16_tflops = run(false);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

}  // namespace xb
