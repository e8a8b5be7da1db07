// FP32-accurate tensor-core GEMM on tcgen05 (3xTF32, TMEM accumulator, TMA).
//
// The float32 configs' products (cfg4/cfg5: Y = A X, Z = A^T Q with A in
// float32, Precision.SINGLE — the reference's f32 compute dtype,
// core.py:43-46) on Blackwell's 5th-generation tensor cores. TF32 alone is
// too coarse for the 1e-3 subspace target, so each product is
// split: a = a_hi + a_lo with a_hi = tf32(a), a_lo = a - a_hi (exact in f32),
// and  A B ~ A_hi B_hi + A_hi B_lo + A_lo B_hi  (three tcgen05.mma.kind::tf32
// into one f32 TMEM accumulator; the dropped A_lo B_lo term is ~2^-22).
//
// Warp roles (704 threads, one CTA per 128 x BN output tile):
//   warp 0      TMA producer: raw A tile + the pre-split B_hi / B_lo tiles,
//               a 3-4 deep shared-memory ring
//   warp 1      TMEM allocator + single-thread MMA issuer
//   warps 2-5   converters: raw A tile -> A_hi, A_lo written straight into
//               TMEM (tcgen05.st; thread = tile row, so for the transposed
//               view of A this is also the transpose). The MMA takes A from
//               TMEM and only B from shared memory: with A in shared memory
//               too, operand reads nearly saturated the shared-memory port and
//               the converted planes limited the ring to 2 stages.
//   warps 6-21  drain + epilogue: 4 warps per TMEM lane quadrant, each owning
//               BN/4 columns of its 32 rows
// Barriers: full[s] (TMA) -> conv[s] (converters; A slot kt % 2 filled) ->
// MMA -> commit empty[s] (stage free) + aempty[kt % 2] (A slot free).
//
// Accumulation: the tensor core's f32 accumulator does not round to nearest
// (measured: the error grows ~linearly with the accumulation chain, e.g. a
// K=65536 product is ~30x less accurate than an f32 round-to-nearest sum), so
// the MMA accumulates only P k-tiles (P*32 of K, XB_TG_DRAIN) into one of two
// TMEM buffers; the drain warps fold each finished group into f32 registers
// with ordinary round-to-nearest adds while the MMA fills the other buffer
// (tmem_full[b] / tmem_empty[b]). The result is as accurate as an f32 SGEMM.
// Split-K slices go to an f64 workspace reduced in slice order by dgemm.cu's
// deterministic reduce.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "tc_util.cuh"

namespace xb {
namespace {
using namespace tc;

constexpr int TBM = 128;  // UMMA_M (cta_group::1)
constexpr int TBK = 32;   // one 128-byte swizzle atom of tf32
constexpr int kDrainGroups = 4;  // column segments per TMEM lane quadrant
constexpr int kThreadsT = 192 + 128 * kDrainGroups;

// tf32 "hi" part: the f32 bit pattern with the 13 low mantissa bits cleared
// (exactly the truncation the tensor core applies to a tf32 operand), so
// hi is bit-exact what the MMA uses and lo = x - hi is exact in f32.
__device__ __forceinline__ uint32_t to_tf32(float x) {
  return __float_as_uint(x) & 0xFFFFE000u;
}

// Shared-memory matrix descriptor: K-major, 128B swizzle, 8-row groups 1024 B
// apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // SBO
  d |= (uint64_t)1 << 46;              // descriptor version
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}

template <int BN>
__device__ __forceinline__ uint32_t idesc_tf32() {
  return (1u << 4)                       // D: f32
         | (2u << 7) | (2u << 10)        // A, B: tf32
         | ((uint32_t)(BN >> 3) << 17)   // N
         | ((uint32_t)(TBM >> 4) << 24);  // M
}


template <int BN>
struct TCfg {
  static constexpr int A_BYTES = TBM * TBK * 4;        // 16 KB raw A tile (TMA destination)
  static constexpr int B_BYTES = BN * TBK * 4;         // BN rows x 128 B per B plane
  static constexpr int B_AL = ((B_BYTES + 1023) / 1024) * 1024;
  static constexpr int RAW = 0;
  static constexpr int BHI = RAW + A_BYTES;
  static constexpr int BLO = BHI + B_AL;
  static constexpr int STAGE = BLO + B_AL;
  static constexpr int STAGES = (200 * 1024) / STAGE > 4 ? 4 : (200 * 1024) / STAGE;
  static constexpr int BAR_OFF = STAGES * STAGE;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;    // + barriers (<= 3 NS + 8 + NS), tmem slot, align slack
  // TMEM columns: two accumulator buffers [0, BN), [BN, 2 BN) (the MMA fills
  // one while the drain warps fold the other), then two A slots of 64
  // columns (A_hi: 32 tf32 columns, A_lo: 32) written by the converters.
  static constexpr int ACOL = 2 * BN;
  static constexpr int USED = ACOL + 2 * 64;
  static constexpr int TMEM_COLS = USED <= 32 ? 32 : USED <= 64 ? 64 : USED <= 128 ? 128 : USED <= 256 ? 256 : 512;
  static constexpr int SEG = BN / kDrainGroups;        // columns per drain thread
  static_assert(USED <= 512, "TMEM: accumulators + A slots exceed 512 columns");
};

__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                            uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

// 16 consecutive TMEM columns of this thread's lane <- v[0..15]
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15])
      : "memory");
}

template <int BN, bool TRANS_A>
__global__ void __launch_bounds__(kThreadsT, 1)
    tgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                 const __grid_constant__ CUtensorMap tmBl, int64_t M, int64_t N, int64_t K,
                 double* __restrict__ C, int64_t ldc, int64_t split_stride, int64_t k_per_split,
                 int accumulate, int drain_tiles, int tiles_n, int tiles_m, int splits,
                 int group_m, int cl) {
  using Cfg = TCfg<BN>;
  constexpr int NS = Cfg::STAGES;
  static_assert(Cfg::SEG % 8 == 0, "drain segment must be a multiple of 8 columns");
  extern __shared__ unsigned char smem_raw_t[];
  // 1024-byte alignment by pointer arithmetic on the shared array, so the
  // compiler keeps shared-space (LDS/STS) accesses
  unsigned char* smem = smem_raw_t + ((1024u - (su32(smem_raw_t) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* conv = full + NS;
  uint64_t* empty = conv + NS;
  uint64_t* aempty = empty + NS;         // [2] TMEM A slot free (MMA commit)
  uint64_t* tmem_full = aempty + 2;      // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint64_t* cempty = tmem_empty + 2;     // [NS] cluster leader: stage free in all cl CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + NS);
  // cluster of cl CTAs = the n-tiles of one (m-tile, split): the leader
  // (rank 0) multicasts the raw A tile to all of them, so A is read once
  // per m-tile from L2/HBM instead of once per n-tile
  const uint32_t crank = cl > 1 ? cluster_ctarank() : 0u;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Raster (1-D grid): n-tile fastest (the CTAs sharing an A tile run
  // together: one HBM read of A), then m-tiles within a group of group_m,
  // then splits, then groups. Co-resident CTAs thus touch only ~group_m x 128
  // rows of A (a wide row-major A has every row in its own 2 MB page; with
  // all m-tiles marching along K together the TLB thrashed: 122 vs 224 TF/s
  // at K = 2^20) while group_m m-tiles still share each B k-tile in L2.
  int64_t L = blockIdx.x;
  const int nt = (int)(L % tiles_n);
  L /= tiles_n;
  const int64_t per_group = (int64_t)group_m * splits;
  const int64_t mg = L / per_group;
  const int64_t w = L - mg * per_group;
  const int gsz = (int)min((int64_t)group_m, (int64_t)tiles_m - mg * group_m);
  const int split = (int)(w / gsz);
  const int64_t mt = mg * group_m + (w - (int64_t)split * gsz);
  const int64_t m0 = mt * TBM;
  const int64_t n0 = (int64_t)nt * BN;
  const int64_t kbeg = (int64_t)split * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  const int ktiles = (int)((kend - kbeg + TBK - 1) / TBK);
  const int P = drain_tiles;
  const int groups = (ktiles + P - 1) / P;
  C += (int64_t)split * split_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&aempty[b], 1);
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4 * kDrainGroups);
    }
    for (int s = 0; s < NS; ++s) mbar_init(&cempty[s], cl);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (cl > 1)
    cluster_sync_all();  // every CTA's barriers initialised before any multicast
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer ------------------------------------------------------
    if (lane == 0) {
      const uint32_t bytes = Cfg::A_BYTES + 2 * Cfg::B_BYTES;
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % NS;
        if (kt >= NS) {
          mbar_wait_park(&empty[s], ((kt / NS) & 1) ^ 1);
          // the leader may refill the A slot only when every CTA freed it
          if (cl > 1 && crank == 0) mbar_wait_park(&cempty[s], ((kt / NS) & 1) ^ 1);
        }
        unsigned char* st = smem + s * Cfg::STAGE;
        const int32_t k0 = (int32_t)(kbeg + (int64_t)kt * TBK);
        mbar_expect_tx(&full[s], bytes);
        const int32_t ca = TRANS_A ? (int32_t)m0 : k0, cb = TRANS_A ? k0 : (int32_t)m0;
        // TRANS_A: [BK][BM] M inner; else [BM][BK] swizzled
        if (cl == 1)
          tma_load_2d(st + Cfg::RAW, &tmA, &full[s], ca, cb);
        else if (crank == 0)
          tma_load_2d_mc(st + Cfg::RAW, &tmA, &full[s], ca, cb, (uint16_t)((1u << cl) - 1));
        // B planes are k-blocked ([K/32][N][32]): one contiguous BN x 128 B tile
        tma_load_3d(st + Cfg::BHI, &tmBh, &full[s], 0, (int32_t)n0, k0 / TBK);
        tma_load_3d(st + Cfg::BLO, &tmBl, &full[s], 0, (int32_t)n0, k0 / TBK);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: A_hi/A_lo from TMEM, B_hi/B_lo from shared memory;
    // group g of P k-tiles accumulates into buffer g & 1 ----------------------
    const uint32_t idesc = idesc_tf32<BN>();
    const uint32_t cempty0 = cl > 1 ? mapa_rank(cempty, 0) : 0u;  // leader's cempty[0]
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % NS, a = kt & 1;
      const int g = kt / P, b = g & 1;
      const bool first = (kt % P) == 0;
      const bool last = (kt % P) == P - 1 || kt == ktiles - 1;
      if (first && g >= 2) mbar_wait(&tmem_empty[b], ((g >> 1) - 1) & 1);
      mbar_wait(&conv[s], (kt / NS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      if (lane == 0) {
        const uint32_t d = tmem + (uint32_t)(b * BN);
        const uint32_t ahi = tmem + (uint32_t)(Cfg::ACOL + a * 64);
        unsigned char* st = smem + s * Cfg::STAGE;
        const uint64_t bh = sw128_desc(su32(st + Cfg::BHI));
        const uint64_t bl = sw128_desc(su32(st + Cfg::BLO));
#pragma unroll
        for (int kk = 0; kk < TBK / 8; ++kk) {
          const uint64_t off = (uint64_t)(kk * 32) >> 4;  // 8 tf32 = 32 B inside the atom
          const uint32_t ah = ahi + (uint32_t)(kk * 8), al = ah + 32;
          mma_tf32_ta(d, ah, bh + off, idesc, (!first || kk > 0) ? 1u : 0u);
          mma_tf32_ta(d, ah, bl + off, idesc, 1u);
          mma_tf32_ta(d, al, bh + off, idesc, 1u);
        }
        mma_commit(&empty[s]);
        if (cl > 1) mma_commit_cluster(cempty0 + (uint32_t)(s * sizeof(uint64_t)));
        mma_commit(&aempty[a]);
        if (last) mma_commit(&tmem_full[b]);
      }
      __syncwarp();
    }
  } else if (warp < 6) {
    // ---- converters: raw A -> A_hi, A_lo in TMEM (lane = tile row) -----------
    // warp w may touch TMEM lanes 32 (w % 4) .. +31: warps 2-5 cover all four
    const int m = 32 * (warp & 3) + lane;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % NS, a = kt & 1;
      mbar_wait_park(&full[s], (kt / NS) & 1);
      if (kt >= 2) mbar_wait_park(&aempty[a], ((kt >> 1) - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const unsigned char* raw = smem + s * Cfg::STAGE + Cfg::RAW;
      const uint32_t tbase = tmem + lane_base + (uint32_t)(Cfg::ACOL + a * 64);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int chunk = half * 4 + c;  // 16-byte chunk = k 4 chunk .. +3
          float4 v;
          if constexpr (!TRANS_A) {
            // [BM][BK] rows of 128 B, 16-byte chunks XOR-swizzled by row % 8
            v = *reinterpret_cast<const float4*>(raw + m * 128 + ((chunk ^ (m & 7)) << 4));
          } else {
            // [BK][BM], M contiguous
            const float* rf = reinterpret_cast<const float*>(raw);
            v.x = rf[(4 * chunk + 0) * TBM + m];
            v.y = rf[(4 * chunk + 1) * TBM + m];
            v.z = rf[(4 * chunk + 2) * TBM + m];
            v.w = rf[(4 * chunk + 3) * TBM + m];
          }
          const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t h = to_tf32(x[e]);
            hi[4 * c + e] = h;
            lo[4 * c + e] = __float_as_uint(x[e] - __uint_as_float(h));
          }
        }
        tmem_st16(tbase + (uint32_t)(half * 16), hi);
        tmem_st16(tbase + (uint32_t)(32 + half * 16), lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
  } else {
    // ---- drain warps: TMEM group partials -> f32 register sums (round to
    // nearest), then the f64 epilogue. Warp w reads TMEM lanes 32 (w % 4) ..
    // +31 (the hardware's lane-quadrant rule) and column segment (w - 6) / 4.
    const int q = warp & 3;
    const int seg = (warp - 6) >> 2;
    const int row = 32 * q + lane;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    float acc[Cfg::SEG];
#pragma unroll
    for (int j = 0; j < Cfg::SEG; ++j) acc[j] = 0.f;
    for (int g = 0; g < groups; ++g) {
      const int b = g & 1;
      mbar_wait_park(&tmem_full[b], (g >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t base = tmem + lane_base + (uint32_t)(b * BN + seg * Cfg::SEG);
#pragma unroll
      for (int c0 = 0; c0 < Cfg::SEG; c0 += 8) {
        uint32_t v[8];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7])
            : "r"(base + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[c0 + j] += __uint_as_float(v[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[b]);
    }
    const int64_t r = m0 + row;
    if (r < M) {
      const int64_t cbase = n0 + seg * Cfg::SEG;
      double* dst = C + r * ldc + cbase;
#pragma unroll
      for (int j = 0; j < Cfg::SEG; ++j) {
        if (cbase + j < N) {
          const double x = (double)acc[j];
          dst[j] = accumulate ? dst[j] + x : x;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  // no CTA leaves while a cluster peer may still multicast into it or
  // arrive on its barriers
  if (cl > 1)
    cluster_sync_all();
  else
    __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(Cfg::TMEM_COLS));
  }
}

// X (K x N row-major f64, ldx) -> hi, lo (f32, k-blocked [Kp/32][N][32]:
// each k-tile of B is one contiguous N x 128 B slab), hi = tf32(x),
// lo = f32(x - hi); rows K..Kp-1 are zero.
__global__ void split_b_kernel(const double* __restrict__ X, int64_t K, int64_t N, int64_t ldx,
                               float* __restrict__ hi, float* __restrict__ lo, int64_t kp) {
  __shared__ double tile[32][33];
  const int64_t k0 = (int64_t)blockIdx.x * 32, n0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t k = k0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && n < N) ? X[k * ldx + n] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < kp) {
      const double x = tile[threadIdx.x][i];
      const float h = __uint_as_float(to_tf32((float)x));
      const int64_t o = ((int64_t)blockIdx.x * N + n) * 32 + threadIdx.x;
      hi[o] = h;
      lo[o] = (float)(x - (double)h);
    }
  }
}

// k-blocked B plane [KB][N][32] f32: dims {32, N, KB}, boxes {32, bn, 1}, 128B swizzle
CUtensorMap make_map_kblocked(const void* base, uint64_t n, uint64_t kb, uint32_t bn) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {(cuuint64_t)TBK, n, kb};
  const cuuint64_t strides[2] = {TBK * 4, n * TBK * 4};
  const cuuint32_t box[3] = {(cuuint32_t)TBK, bn, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  XB_REQUIRE(r == CUDA_SUCCESS, XB_ECUDA, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string(r));
  return m;
}

int pick_tbn(int64_t N) {
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  if (N <= 192) return 192;
  // wide sketches: 3 x 192 covers cfg5's 552 with 4% padding. BN is capped
  // at 192 by TMEM (2 accumulators + 2 A slots <= 512 columns).
  const int64_t w128 = ceil_div(N, 128) * 128, w192 = ceil_div(N, 192) * 192;
  return w192 <= w128 ? 192 : 128;
}

template <int BN, bool TRANS_A>
void launch_t(const CUtensorMap& ta, const CUtensorMap& bh, const CUtensorMap& bl,
              const DGemmArgs& g, int splits, int64_t kps, double* out, int64_t ldo,
              int64_t stride, cudaStream_t st) {
  using Cfg = TCfg<BN>;
  auto kern = tgemm_kernel<BN, TRANS_A>;
  XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int64_t mtiles = ceil_div(g.M, TBM), ntiles = ceil_div(g.N, BN);
  const int acc_here = (splits == 1 && g.accumulate) ? 1 : 0;
  // k-tiles per TMEM accumulation group (XB_TG_DRAIN overrides for sweeps)
  static const int drain = [] {
    const char* e = knob("XB_TG_DRAIN");
    return e ? std::max(1, atoi(e)) : 2;
  }();
  // m-tiles per raster group (XB_TG_GROUP overrides for sweeps)
  static const int group = [] {
    const char* e = knob("XB_TG_GROUP");
    return e ? std::max(1, atoi(e)) : 8;
  }();
  const int64_t total = ntiles * mtiles * splits;
  XB_REQUIRE(total < ((int64_t)1 << 31), XB_EUNSUPPORTED, "tgemm: too many tiles for one launch");
  // TN: the n-tiles of an (m-tile, split) form one cluster sharing the A
  // tile by TMA multicast — cfg5's A^T Q launches read 123-136 GB from DRAM
  // instead of 201-226 GB for a 68.7 GB A, at the same speed. NN keeps
  // independent CTAs: there the B planes dominate the re-reads and the
  // lockstep of a cluster measured 5-10 % slower. XB_TG_CLUSTER: 0 = never,
  // 2 = also NN.
  static const int cluster_mode = [] {
    const char* e = knob("XB_TG_CLUSTER");
    return e ? atoi(e) : 1;
  }();
  const bool want = cluster_mode == 2 || (cluster_mode == 1 && TRANS_A);
  const int cl = (want && ntiles >= 2 && ntiles <= 4) ? (int)ntiles : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)total);
  cfg.blockDim = dim3(kThreadsT);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  XB_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, bh, bl, g.M, g.N, g.K, out, ldo, stride, kps,
                             acc_here, drain, (int)ntiles, (int)mtiles, splits,
                             (int)std::min<int64_t>(group, mtiles), cl));
  check_launch("tgemm");
}

}  // namespace

bool tgemm_supported(const DGemmArgs& g) {
  if (!g.a_f32) return false;
  if ((reinterpret_cast<uintptr_t>(g.A) & 15) != 0 || (g.lda % 4) != 0) return false;
  if (g.M < 1 || g.N < 1 || g.K < 1) return false;
  static const int env = [] {
    const char* e = knob("XB_F32_GEMM");
    return (e && strcmp(e, "dmma") == 0) ? 0 : 1;
  }();
  return env == 1;
}

int tgemm_plan_splits(const DGemmArgs& g) {
  const int bn = pick_tbn(g.N);
  const int64_t tiles = ceil_div(g.M, TBM) * ceil_div(g.N, bn);
  const int64_t kt = ceil_div(g.K, TBK);
  // K per split slice (slices are summed in f64); the TMEM groups inside a
  // slice are summed in f32 registers, so the chain only bounds that f32 sum.
  static const int64_t chain = [] {
    const char* e = knob("XB_TG_CHAIN");
    return e ? std::max<int64_t>(32, atoll(e)) : (int64_t)32768;
  }();
  int s = (int)std::max<int64_t>(1, ceil_div(g.K, chain));
  while (tiles * s < 2 * kNumSMs && kt / (s * 2) >= 8) s *= 2;
  return std::max(1, std::min<int>(s, (int)kt));
}

size_t tgemm_b_floats(const DGemmArgs& g) { return (size_t)g.N * round_up(g.K, TBK); }

void tgemm(const DGemmArgs& g, int splits, double* work, float* bhi, float* blo, cudaStream_t st) {
  const int64_t kp = round_up(g.K, TBK);
  {
    dim3 grid((unsigned)ceil_div(kp, 32), (unsigned)ceil_div(g.N, 32));
    split_b_kernel<<<grid, dim3(32, 8), 0, st>>>(g.B, g.K, g.N, g.ldb, bhi, blo, kp);
    check_launch("split_b");
  }
  splits = std::max(1, std::min<int>(splits, (int)ceil_div(g.K, TBK)));
  const int64_t kps = round_up(ceil_div(g.K, splits), TBK);
  splits = (int)ceil_div(g.K, kps);
  double* out = g.C;
  int64_t ldo = g.ldc, stride = 0;
  if (splits > 1) {
    XB_REQUIRE(work != nullptr, XB_ECUDA, "tgemm: split-K workspace missing");
    out = work;
    ldo = round_up(g.N, 2);
    stride = g.M * ldo;
  }
  const int bn = pick_tbn(g.N);
  // A: NN -> [M][K] K-major, 128B-swizzled boxes {32, 128};
  //    TN -> [K][M] M-contiguous, unswizzled boxes {128, 32} (the converter transposes)
  const CUtensorMap ta = g.trans_a
                             ? make_map(g.A, (uint64_t)g.M, (uint64_t)g.K, g.lda, TBM, TBK, false)
                             : make_map(g.A, (uint64_t)g.K, (uint64_t)g.M, g.lda, TBK, TBM, true);
  const CUtensorMap th = make_map_kblocked(bhi, (uint64_t)g.N, (uint64_t)(kp / TBK), bn);
  const CUtensorMap tl = make_map_kblocked(blo, (uint64_t)g.N, (uint64_t)(kp / TBK), bn);
#define XB_T(BN)                                                                  \
  if (g.trans_a)                                                                  \
    launch_t<BN, true>(ta, th, tl, g, splits, kps, out, ldo, stride, st);         \
  else                                                                            \
    launch_t<BN, false>(ta, th, tl, g, splits, kps, out, ldo, stride, st);        \
  break;
  switch (bn) {
    case 64: XB_T(64)
    case 128: XB_T(128)
    default: XB_T(192)
  }
#undef XB_T
  if (splits > 1) launch_split_reduce(work, g.M, g.N, ldo, stride, splits, g.C, g.ldc, g.accumulate, st);
}

}  // namespace xb
