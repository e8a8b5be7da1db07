// tcgen05.mma.kind::i8 issue patterns on one SM (standalone microbenchmark):
// how many cycles does a sequence of MMAs with given accumulator offsets and
// N take when consecutive MMAs are independent, dependent on the same
// accumulator, or overlap partially as the grouped slice products of
// ozgemm_kernel do? No loads: operands are two fixed shared-memory tiles.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_mma_pattern_bench tools/mma_pattern_bench.cu
//   tools/_mma_pattern_bench
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <vector>

constexpr int kRep = 16;  // pattern repetitions per commit
struct Pattern {
  int n;
  int doff[16];
  int ncol[16];
};
__host__ __device__ constexpr Pattern pattern(int id) {
  switch (id) {
    case 0: return {2, {0, 256}, {256, 256}};
    case 1: return {2, {0, 0}, {256, 256}};
    case 2: return {2, {0, 256}, {128, 128}};
    case 3: return {2, {0, 0}, {128, 128}};
    case 4: return {2, {0, 256}, {64, 64}};
    case 5: return {2, {0, 0}, {64, 64}};
    case 6: return {8, {0, 256, 64, 320, 128, 192, 256, 320}, {256, 128, 256, 64, 256, 192, 128, 64}};
    case 7: return {8, {0, 256, 0, 256, 0, 256, 0, 256}, {256, 128, 256, 64, 256, 192, 128, 64}};
    case 8: return {8, {0, 0, 0, 0, 0, 0, 0, 0}, {256, 128, 256, 64, 256, 192, 128, 64}};
    case 9: return {3, {0, 64, 128}, {256, 256, 256}};
    case 10: return {6, {0, 32, 64, 96, 128, 160}, {224, 192, 160, 128, 96, 64}};
    case 11: return {8, {0, 256, 0, 256, 0, 256, 0, 256}, {256, 256, 256, 256, 256, 256, 256, 256}};
    default: return {8, {0, 0, 64, 64, 128, 128, 192, 192}, {256, 256, 256, 256, 256, 256, 256, 256}};
  }
}
constexpr int kPatterns = 25;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t sbo, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

template <int ID, bool TS = false, int NC = 0, int WR = 0, bool RING = false>
__global__ void __launch_bounds__(128) pattern_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(16) uint8_t wr_ring[];  // WR > 0: 96 KB the other warps write into
  __shared__ volatile int done;
  constexpr Pattern pat = pattern(ID);
  __shared__ __align__(1024) uint8_t a_s[128 * 32];
  __shared__ __align__(1024) uint8_t b_s[256 * 32];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(8) uint64_t scratch[2];  // NC commits per pattern land here, never waited on
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 32 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(a_s)[i] = 0x01010101u * (i & 3);
  for (int i = threadIdx.x; i < 256 * 32 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(b_s)[i] = 0x01010101u * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[1])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&scratch[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&scratch[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        su32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (WR > 0 && warp > 0) {
    // 96 threads store WR KB per 700 cycles (16-byte stores), paced by the clock
    const int t = threadIdx.x - 32;
    const int per_tick = WR * 1024 / 16 / 96;  // stores per thread per tick
    uint4 v = make_uint4(t, t, t, t);
    uint32_t pos = 0;
    long long next = clock64();
    while (!done) {
      for (int i = 0; i < per_tick; ++i) {
        *reinterpret_cast<uint4*>(wr_ring + ((pos + (uint32_t)t) % 6144u) * 16u) = v;
        pos += 96;
      }
      next += 700;
      while (clock64() < next && !done) {
      }
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t idesc0 = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 4) << 24);
    const uint64_t da = smem_desc(su32(a_s), 256, 128);
    const uint64_t db = smem_desc(su32(b_s), 256, 128);
    // two barriers, batch `it` commits to bar[it & 1]; the wait for batch it - 1
    // comes right after the commit of batch it, so no barrier is ever more than
    // one phase ahead of its waiter
    uint32_t phase[2] = {0, 0};
    auto wait = [&](int b) {
      asm volatile(
          "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra W_%=;\n}\n" ::"r"(su32(&bar[b])),
          "r"(phase[b])
          : "memory");
      phase[b] ^= 1;
    };
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
      for (int r = 0; r < kRep; ++r) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                  su32(&scratch[c & 1]))
              : "memory");
#pragma unroll
      for (int j = 0; j < pat.n; ++j) {
        const uint32_t d = tmem + (uint32_t)pat.doff[j];
        const uint32_t idesc = idesc0 | ((uint32_t)(pat.ncol[j] >> 3) << 17);
        if (RING) {
          // operands where ozgemm_kernel keeps them: stage r % 5 of a ring in the
          // dynamic shared memory, left slice t at t * 4096, right slices from
          // 24576 + u0 * 2048 (pattern 6's (t, u0) list)
          constexpr int tt[8] = {0, 0, 1, 1, 2, 3, 4, 5};
          constexpr int uu[8] = {0, 4, 0, 4, 0, 0, 0, 0};
          const uint32_t stg = su32(wr_ring) + (uint32_t)((r % 5) * 36864);
          const uint64_t xa = smem_desc(stg + tt[j % 8] * 4096, 256, 128);
          const uint64_t xb = smem_desc(stg + 24576 + uu[j % 8] * 2048, 256, 128);
          if (TS)
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                "r"(tmem + 448u + 8u * (uint32_t)tt[j % 8]), "l"(xb), "r"(idesc), "r"(1));
          else
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                "l"(xa), "l"(xb), "r"(idesc), "r"(1));
        } else if (TS)  // A operand from TMEM (columns 448..: a 128 x 32-byte slot per slice)
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
              "r"(tmem + 448u + 8u * (uint32_t)(j % 6)), "l"(db), "r"(idesc), "r"(1));
        else
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
              "l"(da), "l"(db), "r"(idesc), "r"(1));
      }
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              su32(&bar[it & 1]))
          : "memory");
      if (it > 0) wait((it - 1) & 1);
    }
    wait((iters - 1) & 1);
    if (blockIdx.x == 0) *cycles = clock64() - t0;
    done = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  const char* names[kPatterns] = {
      "2 x N=256, alternating accumulators (peak)",
      "2 x N=256, SAME accumulator (dependent)",
      "2 x N=128, alternating",
      "2 x N=128, same accumulator",
      "2 x N=64, alternating",
      "2 x N=64, same accumulator",
      "ozgemm S=6 k-tile: (0,256)(256,128)(64,256)(320,64)(128,256)(192,192)(256,128)(320,64)",
      "same N list, accumulators alternating 0 / 256 (no overlap between neighbours)",
      "same N list, all on accumulator 0 (fully dependent)",
      "N=256 x3 shifted by 64 (levels 0-3, 1-4, 2-5)",
      "6 MMAs N=224..64 shifted by 32 (a 32-column-tile variant)",
      "8 x N=256 alternating accumulators",
      "8 x N=256: pairs on the same accumulator, shifted by 64 between pairs",
      "ozgemm S=6 k-tile with the A operand from TMEM (TS mode)",
      "2 x N=256 alternating, A operand from TMEM",
      "ozgemm S=6 k-tile, SS, 1 tcgen05.commit per k-tile",
      "ozgemm S=6 k-tile, SS, 2 commits per k-tile",
      "ozgemm S=6 k-tile, TS, 1 commit per k-tile",
      "ozgemm S=6 k-tile, TS, 2 commits per k-tile",
      "ozgemm S=6 k-tile, SS, other warps store 36 KB per 700 cycles into shared memory",
      "ozgemm S=6 k-tile, SS, other warps store 72 KB per 700 cycles",
      "ozgemm S=6 k-tile, TS, other warps store 24 KB per 700 cycles",
      "ozgemm S=6 k-tile, TS, other warps store 72 KB per 700 cycles",
      "ozgemm S=6 k-tile, SS, operands at the kernel's addresses (5-stage ring, per-slice tiles)",
      "ozgemm S=6 k-tile, TS, right slices at the kernel's addresses",
  };
  long long* dc;
  cudaMalloc(&dc, sizeof(long long));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 1000;
  auto launch = [&](int id) {
    switch (id) {
#define XB_CASE(I) case I: pattern_kernel<I><<<sms, 128>>>(iters, dc); break;
      XB_CASE(0) XB_CASE(1) XB_CASE(2) XB_CASE(3) XB_CASE(4) XB_CASE(5) XB_CASE(6)
      XB_CASE(7) XB_CASE(8) XB_CASE(9) XB_CASE(10) XB_CASE(11) XB_CASE(12)
#undef XB_CASE
      case 13: pattern_kernel<6, true><<<sms, 128>>>(iters, dc); break;
      case 14: pattern_kernel<0, true><<<sms, 128>>>(iters, dc); break;
      case 15: pattern_kernel<6, false, 1><<<sms, 128>>>(iters, dc); break;
      case 16: pattern_kernel<6, false, 2><<<sms, 128>>>(iters, dc); break;
      case 17: pattern_kernel<6, true, 1><<<sms, 128>>>(iters, dc); break;
      case 18: pattern_kernel<6, true, 2><<<sms, 128>>>(iters, dc); break;
#define XB_WR(I, TSV, KB)                                                                      \
  case I:                                                                                      \
    cudaFuncSetAttribute(pattern_kernel<6, TSV, 1, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         98304);                                                               \
    pattern_kernel<6, TSV, 1, KB><<<sms, 128, 98304>>>(iters, dc);                             \
    break;
      XB_WR(19, false, 36) XB_WR(20, false, 72) XB_WR(21, true, 24) XB_WR(22, true, 72)
#undef XB_WR
      case 23:
        cudaFuncSetAttribute(pattern_kernel<6, false, 1, 0, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 36864);
        pattern_kernel<6, false, 1, 0, true><<<sms, 128, 5 * 36864>>>(iters, dc);
        break;
      case 24:
        cudaFuncSetAttribute(pattern_kernel<6, true, 1, 0, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 36864);
        pattern_kernel<6, true, 1, 0, true><<<sms, 128, 5 * 36864>>>(iters, dc);
        break;
    }
  };
  for (int id = 0; id < kPatterns; ++id) {
    const Pattern p = pattern(id == 14 ? 0 : id >= 13 ? 6 : id);
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      launch(id);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error: %s\n", cudaGetErrorString(e));
        return 1;
      }
      long long c = 0;
      cudaMemcpy(&c, dc, sizeof(c), cudaMemcpyDeviceToHost);
      best = best < (double)c / iters / kRep ? best : (double)c / iters / kRep;
    }
    int ideal = 0;
    for (int j = 0; j < p.n; ++j) ideal += p.ncol[j] / 2;
    printf("%7.1f cycles per pattern (ideal %4d, %5.1f %% of peak)  %s\n", best, ideal,
           100.0 * ideal / best, names[id]);
    fflush(stdout);
  }
  return 0;
}
