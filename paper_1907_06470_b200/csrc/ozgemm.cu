// FP64 products on the int8 tensor cores (tcgen05.mma.kind::i8): an
// Ozaki-scheme split of both operands into S signed 8-bit digit slices with
// power-of-two row / column scales, exact int32 slice products, and an f64
// recombination in the epilogue.
//
// FP64 has no tcgen05 kind on sm_100a; the legacy DMMA path (mma.sync.f64,
// dgemm.cu) peaks at ~37 TF/s. The int8 tensor pipe runs ~120x faster, so
// the S(S+1)/2 slice products (21 for S = 6) still leave a several-fold
// margin. Numerics (t, u, d 0-based): with row scale 2^e_i (|L_ik| 2^-e_i
// < 126/128) and column scale 2^f_j,
//     L_ik = 2^e_i sum_t a_t,ik 2^-(7+8t) + r_ik,   |r_ik| <= 2^(e_i-8S)
// (a_0 in [-127, 127], balanced a_t in [-128, 127] below: 7 + 8 (S-1) = 47
// bits at S = 6, round to nearest), and
//     (L R)_ij = 2^(e_i+f_j) sum_{d<S} 2^-(14+8d) sum_{t+u=d} (a_t b_u)_ij
// (pairs with t + u >= S are dropped: below 2^-8S of the row/column scale).
// Every (a_t b_u) is exact in int32 while K_chunk * 2^14 * (pairs per level
// <= S) < 2^31, i.e. K_chunk <= 16384; longer reductions are split over K
// into f64 slices summed in slice order. The error is relative to the
// row/column max-norm scale, so the engine keeps matrices whose rows or
// columns span more than 64x their RMS on DMMA (row_exp / col_exp guard).
//
// Layout: left operand slices L[t] (k-blocked [kp/32][rows_p][32] int8: each
// 128-row k-tile is contiguous) with row exponents; right operand slices R[u] (np x kp int8, K contiguous: the
// transposed right matrix) with column exponents. For Y = A X the left
// slices are A's rows (made once per factorisation); for Z = A^T Q they are
// A's columns (a transposed slice set, also made once), so both products run
// the same NN kernel with K-major operands (kind::i8 has no MN-major mode).
//
// Kernel (one CTA per 128 x 48 output tile, 448 threads):
//   warp 0      TMA producer: the S right-slice tiles (48 x 32 B each,
//               32-byte swizzle) of each k-tile, an 8-deep ring
//   warp 1      TMEM allocator + single-thread MMA issuer: per k-tile the
//               S(S+1)/2 pairs (t, u) accumulate into level d = t + u - 2
//               (S int32 accumulators of 48 columns; 4 TMEM A slots)
//   warps 2-13  loaders (3 per TMEM lane quadrant): each thread owns one tile
//               row; it reads its 32-byte row segment of 2 left slices
//               straight from global memory (6 k-tiles in flight in
//               registers) and stores them into a
//               TMEM A slot (tcgen05.st) -- the MMA takes A from TMEM, so
//               shared memory only carries the right slices (an SS-mode A
//               would need ~190 B/clk of shared-memory reads). Then the
//               epilogue: per level tcgen05.ld, int32 -> f64, * 2^-7d, sum,
//               * 2^(e_i + f_j), store (or += / split-K slice).
#include <algorithm>

#include "common.cuh"
#include "tc_util.cuh"

namespace xb {
namespace {
using namespace tc;

constexpr int OBM = 128;   // UMMA_M
constexpr int OBN = 64;    // UMMA_N (S levels x 64 TMEM columns + 2 A slots fit in 512)
constexpr int OBK = 32;    // int8 K per MMA = one 32-byte swizzle row
constexpr int OEPIW = 4;   // epilogue warps (one TMEM lane quadrant each)
constexpr int OTHREADS = 64 + 32 * OEPIW;

template <int S>
struct OCfg {
  static constexpr int ATILE = OBM * OBK;            // 4 KB: one left slice of a k-tile
  static constexpr int RTILE = OBN * OBK;            // 2 KB: one right slice
  static constexpr int STAGE = S * (ATILE + RTILE);
  static constexpr int NS = (200 * 1024) / STAGE;    // ring depth (5 at S = 6)
  static constexpr int BAR_OFF = NS * STAGE;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int ACC_COLS = S * OBN;           // level accumulators
  static constexpr int ASLOT = S * (OBK / 4);        // TMEM columns per A slot
  static constexpr int USED = ACC_COLS + 2 * ASLOT;
  static constexpr int TMEM_COLS = USED <= 256 ? 256 : 512;
  static_assert(USED <= 512, "TMEM budget");
};

template <int S>
__device__ __forceinline__ uint32_t idesc_i8() {
  return (2u << 4)                          // D: s32
         | (1u << 7) | (1u << 10)           // A, B: signed 8-bit
         | ((uint32_t)(OBN >> 3) << 17)     // N
         | ((uint32_t)(OBM >> 4) << 24);    // M
}

// Issued by the whole MMA warp with warp-uniform operands (so they live in
// uniform registers: no per-instruction uniformisation loop); elect.sync
// picks the one lane that issues.
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// smem (128 rows x 32 B, 32-byte swizzle) -> TMEM lanes 0-127, 8 columns
__device__ __forceinline__ void cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n"
      "}\n" ::"r"(taddr),
      "l"(sdesc));
}

__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(su32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4, %5}], [%6];\n" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(bar))
      : "memory");
}

template <int S>
__global__ void __launch_bounds__(OTHREADS, 1)
    ozgemm_kernel(const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmR,
                  const int32_t* __restrict__ eL, const int32_t* __restrict__ eR, int64_t M,
                  int64_t N, int64_t K, double* __restrict__ C, int64_t ldc, int64_t split_stride,
                  int64_t k_per_split, int accumulate, int tiles_n) {
  using Cfg = OCfg<S>;
  constexpr int NS = Cfg::NS;
  extern __shared__ unsigned char smem_raw_o[];
  unsigned char* smem = smem_raw_o + ((1024u - (su32(smem_raw_o) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty = full + NS;
  uint64_t* tmem_full = empty + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (int)(blockIdx.x % tiles_n);
  const int64_t mt = blockIdx.x / tiles_n;
  const int64_t m0 = mt * OBM, n0 = (int64_t)nt * OBN;
  const int64_t kbeg = (int64_t)blockIdx.y * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  const int ktiles = kend > kbeg ? (int)((kend - kbeg + OBK - 1) / OBK) : 0;
  C += (int64_t)blockIdx.y * split_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(tmem_slot)),
                 "n"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer: S left-slice tiles (4-D box over the k-blocked
    // slices) and S right-slice tiles per k-tile ------------------------------
    if (lane == 0) {
      const int32_t kb0 = (int32_t)(kbeg / OBK);
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % NS;
        if (kt >= NS) mbar_wait_park(&empty[s], ((kt / NS) & 1) ^ 1);
        unsigned char* st = smem + s * Cfg::STAGE;
        mbar_expect_tx(&full[s], Cfg::STAGE);
        tma_load_4d(st, &tmL, &full[s], 0, (int32_t)m0, kb0 + kt, 0);
        tma_load_3d(st + S * Cfg::ATILE, &tmR, &full[s], (int32_t)(kbeg + (int64_t)kt * OBK),
                    (int32_t)n0, 0);
      }
    }
  } else if (warp == 1) {
    // ---- MMA warp: tcgen05.cp of the left slices into a TMEM A slot, then
    // the S(S+1)/2 slice products (cp and mma run in issue order) -------------
    const uint32_t idesc = idesc_i8<S>();
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t sbase = su32(smem);
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % NS, a = kt & 1;
      mbar_wait(&full[s], (kt / NS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t aslot = tm + (uint32_t)(Cfg::ACC_COLS + a * Cfg::ASLOT);
      const uint32_t abase = sbase + (uint32_t)(s * Cfg::STAGE);
      const uint32_t rbase = abase + (uint32_t)(S * Cfg::ATILE);
#pragma unroll
      for (int t = 0; t < S; ++t)
        cp_128x256b(aslot + (uint32_t)(t * (OBK / 4)), smem_desc(abase + t * Cfg::ATILE, 256, 6));
      const uint32_t first = kt > 0 ? 1u : 0u;
#pragma unroll
      for (int t = 0; t < S; ++t) {
#pragma unroll
        for (int u = 0; u < S - t; ++u) {
          const int d = t + u;  // level (t + 1) + (u + 1) - 2
          mma_i8(tm + (uint32_t)(d * OBN), aslot + (uint32_t)(t * (OBK / 4)),
                 smem_desc(rbase + u * Cfg::RTILE, 256, 6), idesc, t > 0 ? 1u : first);
        }
      }
      commit_elect(&empty[s]);
      if (kt == ktiles - 1) commit_elect(tmem_full);
      __syncwarp();
    }
  } else {
    // ---- epilogue: levels -> f64, * 2^-7d, sum, * 2^(e_i + f_j), store ----------
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const int64_t grow = m0 + row;
    const bool rvalid = grow < M;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    if (ktiles > 0) {
      mbar_wait_park(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    const int er = rvalid ? eL[grow] : 0;
    double* dst = C + (rvalid ? grow : 0) * ldc;
#pragma unroll 1
    for (int c0 = 0; c0 < OBN; c0 += 16) {
      double acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0;
      if (ktiles > 0) {
#pragma unroll 1
        for (int d = 0; d < S; ++d) {
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
              "%11, %12, %13, %14, %15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tmem + lane_base + (uint32_t)(d * OBN + c0)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          const double sc = ldexp(1.0, -14 - 8 * d);  // level d weight
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = fma((double)(int)v[j], sc, acc[j]);
        }
      }
      if (rvalid) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t col = n0 + c0 + j;
          if (col < N) {
            const double x = scalbn(acc[j], er + eR[col]);
            dst[col] = accumulate ? dst[col] + x : x;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(Cfg::TMEM_COLS));
  }
}

// ---- slicing ---------------------------------------------------------------------

// exponent e with 128 m 2^-e < 126 (the top digit stays within int8 after
// the lower balanced digits borrow from it)
__device__ __forceinline__ int slice_exp(double m) {
  if (!(m > 0.0)) return 0;
  int e = ilogb(m) + 1;  // m 2^-e in [0.5, 1)
  if (scalbn(m, 7 - e) >= 126.0) ++e;
  return e;
}

// Digits of x 2^-e rounded to 7 + 8 (S-1) bits: V = rint(x 2^(7 + 8(S-1) - e))
// = sum_t a_t 2^(8(S-1-t)), a_0 in [-127, 127] (top, weight 2^-7) and
// balanced a_t in [-128, 127] below (weight 2^-(7 + 8t)).
// 2^k as a double (exact for normal k; the slicing scales are far inside)
__device__ __forceinline__ double pow2(int k) {
  return __longlong_as_double((long long)(1023 + max(-1022, min(1023, k))) << 52);
}

template <int S>
__device__ __forceinline__ void slice_digits(double x, int e, int (&a)[S]) {
  const long long v = __double2ll_rn(x * pow2(7 + 8 * (S - 1) - e));
  // balanced base-256 digits without a carry chain: adding 128 at every lower
  // digit position makes them plain bytes u_t (a_t = u_t - 128, i.e. the
  // byte with its top bit flipped); the top digit is what remains above
  constexpr unsigned long long kBias = 0x8080808080ULL >> (8 * (6 - S));
  const unsigned long long u = (unsigned long long)v + kBias;
  a[0] = (int)((long long)u >> (8 * (S - 1)));
#pragma unroll
  for (int t = 1; t < S; ++t)
    a[t] = (int)(int8_t)(uint8_t)(((u >> (8 * (S - 1 - t))) & 0xFF) ^ 0x80);
}

// max |x| over each row (one warp per row) -> slice exponent. The slices
// carry a fixed number of bits relative to the row maximum, so a row whose
// maximum towers over its RMS (max^2 > kOzRange^2 * mean square) loses
// relative accuracy; such matrices raise *wide and stay on DMMA.
constexpr double kOzRange = 64.0;

__global__ void row_exp_kernel(const double* __restrict__ X, int64_t rows, int64_t cols,
                               int64_t ldx, int32_t* __restrict__ e, int* __restrict__ wide) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  const double* r = X + w * ldx;
  double m = 0.0, ss = 0.0;
  for (int64_t c = lane; c < cols; c += 32) {
    const double v = r[c];
    m = fmax(m, fabs(v));
    ss = fma(v, v, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if (lane == 0) {
    e[w] = slice_exp(m);
    if (wide && m * m > kOzRange * kOzRange * (ss / (double)cols)) atomicOr(wide, 1);
  }
}

// max |x| and sum of squares over each column: per-block partials, atomicMax
// on the bit pattern (order-preserving for non-negative doubles); the sums
// only feed the range guard (order does not matter for a threshold test)
__global__ void col_max_kernel(const double* __restrict__ X, int64_t rows, int64_t cols,
                               int64_t ldx, unsigned long long* __restrict__ cmax,
                               double* __restrict__ css) {
  const int64_t c = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * 256;
  if (c >= cols) return;
  double m = 0.0, ss = 0.0;
  for (int64_t r = r0 + threadIdx.y; r < min(rows, r0 + 256); r += blockDim.y) {
    const double v = X[r * ldx + c];
    m = fmax(m, fabs(v));
    ss = fma(v, v, ss);
  }
  atomicMax(cmax + c, (unsigned long long)__double_as_longlong(m));
  if (css) atomicAdd(css + c, ss);
}

__global__ void col_exp_kernel(const unsigned long long* __restrict__ cmax,
                               const double* __restrict__ css, int64_t rows, int64_t cols,
                               int32_t* __restrict__ e, int* __restrict__ wide) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const double m = __longlong_as_double((long long)cmax[c]);
  e[c] = slice_exp(m);
  if (wide && css && m * m > kOzRange * kOzRange * (css[c] / (double)rows)) atomicOr(wide, 1);
}

template <int S>
__device__ __forceinline__ void slice7(double x, int e, int8_t* out, int64_t plane) {
  int a[S];
  slice_digits<S>(x, e, a);
#pragma unroll
  for (int t = 0; t < S; ++t) out[t * plane] = (int8_t)a[t];
}

// row slices, k-blocked: X (rows x cols, ldx) -> P[t][kp/32][rows_p][32],
// zero padded; one thread per 8 consecutive k of a row (8-byte stores)
template <int S>
__global__ void slice_rows_kernel(const double* __restrict__ X, int64_t rows, int64_t cols,
                                  int64_t ldx, const int32_t* __restrict__ e,
                                  int8_t* __restrict__ P, int64_t rows_p, int64_t kp) {
  const int64_t plane = rows_p * kp;
  const int64_t total = plane / 8;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx & 3);
    const int64_t rk = idx >> 2;
    const int64_t r = rk % rows_p, kb = rk / rows_p;
    const int64_t c0 = kb * 32 + j * 8;
    uint64_t w[S];
#pragma unroll
    for (int t = 0; t < S; ++t) w[t] = 0;
    if (r < rows) {
      const int er = e[r];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t c = c0 + q;
        int a[S];
        slice_digits<S>(c < cols ? X[r * ldx + c] : 0.0, er, a);
#pragma unroll
        for (int t = 0; t < S; ++t) w[t] |= (uint64_t)(uint8_t)(int8_t)a[t] << (8 * q);
      }
    }
    int8_t* out = P + (kb * rows_p + r) * 32 + j * 8;
#pragma unroll
    for (int t = 0; t < S; ++t) *reinterpret_cast<uint64_t*>(out + t * plane) = w[t];
  }
}

// column slices, transposed: X (rows x cols) -> P[t] scaled per column, as
// (KBLOCK) [rows_p/32][cols_p][32] or (plain) [cols_p][rows_p]; 32 x 32
// tiles through shared memory
template <int S, bool KBLOCK>
__global__ void slice_cols_t_kernel(const double* __restrict__ X, int64_t rows, int64_t cols,
                                    int64_t ldx, const int32_t* __restrict__ e,
                                    int8_t* __restrict__ P, int64_t cols_p, int64_t rows_p) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? X[r * ldx + c] : 0.0;
  }
  __syncthreads();
  const int64_t plane = cols_p * rows_p;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols_p && r < rows_p) {
      const int ec = c < cols ? e[c] : 0;
      const int64_t o = KBLOCK ? ((r >> 5) * cols_p + c) * 32 + (r & 31) : c * rows_p + r;
      slice7<S>(tile[threadIdx.x][i], ec, P + o, plane);
    }
  }
}

// Both left-operand slice sets of A in one pass (one read of A): the row
// slices [S][kpn/32][mp][32] (row exponents, for Y = A X) and the column
// slices [S][kpm/32][np][32] (column exponents, for Z = A^T Q). A 32 x 32
// tile of A is one k-block of either layout, so each thread packs 4
// consecutive bytes and a tile's writes are 1 KB contiguous per slice.
template <int S>
__global__ void __launch_bounds__(256)
    slice_both_kernel(const double* __restrict__ X, int64_t m, int64_t n, int64_t ldx,
                      const int32_t* __restrict__ er, const int32_t* __restrict__ ec,
                      int8_t* __restrict__ PR, int64_t mp, int64_t kpn, int8_t* __restrict__ PC,
                      int64_t np, int64_t kpm) {
  __shared__ double tile[32][33];
  __shared__ int ser[32], sec[32];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y, t = ty * 32 + tx;
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    tile[i][tx] = (r < m && c < n) ? X[r * ldx + c] : 0.0;
  }
  if (ty == 0) {
    ser[tx] = (r0 + tx < m) ? er[r0 + tx] : 0;
    sec[tx] = (c0 + tx < n) ? ec[c0 + tx] : 0;
  }
  __syncthreads();
  const int a = t >> 3, b4 = (t & 7) * 4;
  if (r0 < mp && c0 < kpn) {  // row layout: (row a, cols b4..b4+3)
    const int64_t planeR = mp * kpn;
    uint32_t w[S];
#pragma unroll
    for (int q = 0; q < S; ++q) w[q] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int d[S];
      slice_digits<S>(tile[a][b4 + j], ser[a], d);
#pragma unroll
      for (int q = 0; q < S; ++q) w[q] |= (uint32_t)(uint8_t)(int8_t)d[q] << (8 * j);
    }
    int8_t* o = PR + ((c0 >> 5) * mp + r0 + a) * 32 + b4;
#pragma unroll
    for (int q = 0; q < S; ++q) *reinterpret_cast<uint32_t*>(o + q * planeR) = w[q];
  }
  if (c0 < np && r0 < kpm) {  // column layout: (col a, rows b4..b4+3)
    const int64_t planeC = np * kpm;
    uint32_t w[S];
#pragma unroll
    for (int q = 0; q < S; ++q) w[q] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int d[S];
      slice_digits<S>(tile[b4 + j][a], sec[a], d);
#pragma unroll
      for (int q = 0; q < S; ++q) w[q] |= (uint32_t)(uint8_t)(int8_t)d[q] << (8 * j);
    }
    int8_t* o = PC + ((r0 >> 5) * np + c0 + a) * 32 + b4;
#pragma unroll
    for (int q = 0; q < S; ++q) *reinterpret_cast<uint32_t*>(o + q * planeC) = w[q];
  }
}

template <int S>
void launch_oz(const CUtensorMap& tl, const CUtensorMap& tr, const int32_t* eL, const int32_t* eR,
               int64_t M, int64_t N, int64_t K, double* out, int64_t ldo, int64_t stride,
               int64_t kps, int splits, int acc, cudaStream_t st) {
  using Cfg = OCfg<S>;
  auto kern = ozgemm_kernel<S>;
  XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int64_t tn = ceil_div(N, OBN), tm = ceil_div(M, OBM);
  XB_REQUIRE(tn * tm < ((int64_t)1 << 31) && splits < 65536, XB_EUNSUPPORTED,
             "ozgemm: grid too large");
  dim3 grid((unsigned)(tn * tm), (unsigned)splits);
  kern<<<grid, OTHREADS, Cfg::SMEM, st>>>(tl, tr, eL, eR, M, N, K, out, ldo, stride, kps, acc,
                                          (int)tn);
  check_launch("ozgemm");
}

// k-blocked left slices [S][kp/32][rows_p][32]: dims {32, rows_p, kb, S},
// boxes {32, 128, 1, S} (one 24 KB load per k-tile), 32-byte swizzle
CUtensorMap make_map_left(const int8_t* base, uint64_t rows_p, uint64_t kb, int S) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {32, rows_p, kb, (cuuint64_t)S};
  const cuuint64_t strides[3] = {32, rows_p * 32, kb * rows_p * 32};
  const cuuint32_t box[4] = {32, (cuuint32_t)OBM, 1, (cuuint32_t)S};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  XB_REQUIRE(r == CUDA_SUCCESS, XB_ECUDA, "cuTensorMapEncodeTiled (left slices) failed: " + std::to_string(r));
  return m;
}

CUtensorMap make_map_slices(const int8_t* base, uint64_t kp, uint64_t np, int S) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {kp, np, (cuuint64_t)S};
  const cuuint64_t strides[2] = {kp, kp * np};
  const cuuint32_t box[3] = {(cuuint32_t)OBK, (cuuint32_t)OBN, (cuuint32_t)S};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3,
                           const_cast<int8_t*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  XB_REQUIRE(r == CUDA_SUCCESS, XB_ECUDA, "cuTensorMapEncodeTiled (slices) failed: " + std::to_string(r));
  return m;
}

}  // namespace

int oz_slices() {
  static const int s = [] {
    const char* e = getenv("XB_OZ_SLICES");
    return e ? std::max(3, std::min(6, atoi(e))) : 6;
  }();
  return s;
}

bool oz_enabled() {
  static const bool on = [] {
    const char* e = getenv("XB_F64_GEMM");
    return !(e && strcmp(e, "dmma") == 0);
  }();
  return on;
}

void oz_row_exp(const double* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* e, int* wide,
                cudaStream_t st) {
  if (rows <= 0) return;
  row_exp_kernel<<<(unsigned)ceil_div(rows * 32, 256), 256, 0, st>>>(X, rows, cols, ldx, e, wide);
  check_launch("row_exp");
}

void oz_col_exp(const double* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* e,
                unsigned long long* scratch, int* wide, cudaStream_t st) {
  if (cols <= 0) return;
  // scratch: cols max words, then (when wide != nullptr) cols sums
  double* css = wide ? reinterpret_cast<double*>(scratch + cols) : nullptr;
  XB_CUDA(cudaMemsetAsync(scratch, 0, (wide ? 2 : 1) * cols * sizeof(unsigned long long), st));
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)std::max<int64_t>(1, ceil_div(rows, 256)));
  col_max_kernel<<<grid, dim3(32, 8), 0, st>>>(X, rows, cols, ldx, scratch, css);
  check_launch("col_max");
  col_exp_kernel<<<(unsigned)ceil_div(cols, 256), 256, 0, st>>>(scratch, css, rows, cols, e, wide);
  check_launch("col_exp");
}

#define OZ_DISPATCH(S, CALL) \
  switch (S) {               \
    case 3: CALL(3); break;  \
    case 4: CALL(4); break;  \
    case 5: CALL(5); break;  \
    default: CALL(6); break; \
  }

void oz_slice_rows(const double* X, int64_t rows, int64_t cols, int64_t ldx, const int32_t* e,
                   int8_t* P, int64_t rows_p, int64_t kp, int S, cudaStream_t st) {
  XB_REQUIRE(kp % 32 == 0, XB_EUNSUPPORTED, "oz_slice_rows: kp % 32");
  const int blocks = (int)std::min<int64_t>(ceil_div(rows_p * kp / 8, 256), kNumSMs * 16);
#define OZ_SR(SS) slice_rows_kernel<SS><<<blocks, 256, 0, st>>>(X, rows, cols, ldx, e, P, rows_p, kp)
  OZ_DISPATCH(S, OZ_SR)
#undef OZ_SR
  check_launch("slice_rows");
}

void oz_slice_cols_t(const double* X, int64_t rows, int64_t cols, int64_t ldx, const int32_t* e,
                     int8_t* P, int64_t cols_p, int64_t rows_p, int S, bool kblocked,
                     cudaStream_t st) {
  dim3 grid((unsigned)ceil_div(rows_p, 32), (unsigned)ceil_div(cols_p, 32));
#define OZ_SC(SS)                                                                             \
  if (kblocked)                                                                               \
    slice_cols_t_kernel<SS, true><<<grid, dim3(32, 8), 0, st>>>(X, rows, cols, ldx, e, P,     \
                                                                cols_p, rows_p);              \
  else                                                                                        \
    slice_cols_t_kernel<SS, false><<<grid, dim3(32, 8), 0, st>>>(X, rows, cols, ldx, e, P,    \
                                                                 cols_p, rows_p)
  OZ_DISPATCH(S, OZ_SC)
#undef OZ_SC
  check_launch("slice_cols_t");
}

void oz_slice_both(const double* X, int64_t m, int64_t n, int64_t ldx, const int32_t* er,
                   const int32_t* ec, int8_t* PR, int64_t mp, int64_t kpn, int8_t* PC, int64_t np,
                   int64_t kpm, int S, cudaStream_t st) {
  XB_REQUIRE(mp % 32 == 0 && np % 32 == 0 && kpn % 32 == 0 && kpm % 32 == 0 && mp >= kpm &&
                 np >= kpn && ceil_div(np, 32) < 65536,
             XB_EUNSUPPORTED, "oz_slice_both: layout");
  dim3 grid((unsigned)(mp / 32), (unsigned)(np / 32));
#define OZ_SB(SS) \
  slice_both_kernel<SS><<<grid, dim3(32, 8), 0, st>>>(X, m, n, ldx, er, ec, PR, mp, kpn, PC, np, kpm)
  OZ_DISPATCH(S, OZ_SB)
#undef OZ_SB
  check_launch("slice_both");
}

int oz_plan_splits(int64_t K) { return (int)std::max<int64_t>(1, ceil_div(K, 16384)); }

void ozgemm(const int8_t* L, int64_t rows_p, int64_t kp, const int32_t* eL, const int8_t* R,
            int64_t np, const int32_t* eR, int64_t M, int64_t N, int64_t K, double* C, int64_t ldc,
            bool accumulate, int S, double* work, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  XB_REQUIRE(kp % 32 == 0 && rows_p >= M, XB_EUNSUPPORTED, "ozgemm: slice layout");
  XB_REQUIRE(rows_p % OBM == 0, XB_EUNSUPPORTED, "ozgemm: rows_p % 128");
  const CUtensorMap tl = make_map_left(L, (uint64_t)rows_p, (uint64_t)(kp / OBK), S);
  const CUtensorMap tr = make_map_slices(R, (uint64_t)kp, (uint64_t)np, S);
  int splits = oz_plan_splits(K);
  const int64_t kps = round_up(ceil_div(K, splits), OBK);
  splits = (int)ceil_div(K, kps);
  double* out = C;
  int64_t ldo = ldc, stride = 0;
  if (splits > 1) {
    XB_REQUIRE(work != nullptr, XB_ECUDA, "ozgemm: split-K workspace missing");
    out = work;
    ldo = round_up(N, 2);
    stride = M * ldo;
  }
  const int acc = (splits == 1 && accumulate) ? 1 : 0;
#define OZ_RUN(SS) launch_oz<SS>(tl, tr, eL, eR, M, N, K, out, ldo, stride, kps, splits, acc, st)
  OZ_DISPATCH(S, OZ_RUN)
#undef OZ_RUN
  if (splits > 1) launch_split_reduce(work, M, N, ldo, stride, splits, C, ldc, accumulate, st);
}

size_t oz_workspace_doubles(int64_t M, int64_t N, int64_t K) {
  const int s = oz_plan_splits(K);
  return s > 1 ? (size_t)s * M * round_up(N, 2) : 0;
}

}  // namespace xb
