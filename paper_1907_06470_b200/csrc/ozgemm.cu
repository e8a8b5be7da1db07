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
// columns span more than 64x their RMS on DMMA (the rc_stats range guard).
//
// Layout (il_off): every operand is stored in HBM exactly as the MMA reads
// it from shared memory — per (k-block of 32, row tile) the S slices are S
// consecutive tiles of rows x 32 bytes in no-swizzle K-major core matrices —
// so each k-tile arrives with ONE linear bulk copy per operand. Left slices
// (128-row tiles) carry per-row exponents, right slices (64-row tiles of the
// transposed right operand) per-column exponents. For Y = A X the left
// slices are A's rows, for Z = A^T Q A's columns (both made once per
// factorisation by slice_both_kernel from one read of A); kind::i8 has no
// MN-major mode, hence the two sets.
//
// Kernel (one CTA per 128 x 64 output tile, 192 threads, 1 CTA per SM):
//   warp 0      producer: per k-tile one bulk copy of the S left slices and
//               one of the S right slices into a ring of NS stages
//   warp 1      TMEM allocator + MMA issuer: the S(S+1)/2 pairs (t, u),
//               t + u < S, accumulate into level d = t + u (S int32
//               accumulators of 64 columns), grouped 4 right slices per MMA,
//               both operands from shared memory (optionally the left slices
//               staged in a TMEM A slot by tcgen05.cp, XB_OZ_TC);
//               tcgen05.commit frees the stage
//   warps 2-5   epilogue (one TMEM lane quadrant each): per level
//               tcgen05.ld, int32 -> f64, * 2^-(14+8d), sum, * 2^(e_i + f_j),
//               store (or += / split-K slice)
#include <algorithm>
#include <cfloat>

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
  static constexpr int SMEM = BAR_OFF + 512 + 1024;  // barriers (3 NS + 1) + TMEM slot, align slack
  static constexpr int ACC_COLS = S * OBN;           // level accumulators
  static constexpr int ASLOT = S * (OBK / 4);        // TMEM columns per A slot
  // (the two TMEM A slots exist only for the tcgen05.cp variants, S <= 6)
  static constexpr int USED = ACC_COLS + (S <= 6 ? 2 * ASLOT : 0);
  static constexpr int TMEM_COLS = USED <= 256 ? 256 : 512;
  static_assert(USED <= 512, "TMEM budget");
};

// Slice layout in HBM = the layout the MMA / tcgen05.cp read from shared
// memory, so each k-tile arrives with ONE linear bulk copy per operand
// (TMA tensor boxes of 32-byte rows ran ~1 request per row: the copies, not
// the tensor pipe, bounded the kernel at 2.6 ms for cfg2's products). For
// row tiles of TR rows x 32 bytes of K: no-swizzle K-major core matrices of
// 8 rows x 16 B (128 B each), the two K-chunks 128 B apart (LBO), 8-row
// groups 256 B apart (SBO); the S slices of one (k-block, row tile) are
// consecutive TR x 32 B tiles.
template <int TR>
__device__ __forceinline__ int64_t il_off(int64_t row, int64_t k, int t, int S, int64_t rows_p) {
  const int64_t kb = k >> 5;
  const int kc = (int)((k >> 4) & 1), kin = (int)(k & 15);
  const int64_t tile = kb * (rows_p / TR) + row / TR;
  const int rr = (int)(row % TR);
  return (tile * S + t) * (TR * 32) + ((rr >> 3) * 2 + kc) * 128 + (rr & 7) * 16 + kin;
}

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

// One lane of the warp, chosen once per k-tile; the raw issue helpers below
// are then called by that lane alone (one elect per k-tile instead of one
// per instruction: the per-instruction elect/vote/uniformise sequence made
// the MMA warp's issue loop, not the tensor pipe, the bound)
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(e));
  return e != 0;
}

__device__ __forceinline__ void mma_i8_1(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void cp_128x256b_1(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;\n" ::"r"(taddr), "l"(sdesc));
}

__device__ __forceinline__ void commit_1(uint32_t cbar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(cbar)
      : "memory");
}

// A from shared memory (descriptor) instead of TMEM
__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
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

// commit arriving on a barrier given by its shared::cluster address
__device__ __forceinline__ void commit_elect_cluster(uint32_t cbar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(cbar)
      : "memory");
}

// 1-D bulk copy multicast to the CTAs of `mask` (same shared offset, each
// completing on its own barrier at the same offset)
__device__ __forceinline__ void bulk_load_mc(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
      "[%1], %2, [%3], %4;\n" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "h"(mask)
      : "memory");
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



// All slice-pair MMAs of one k-tile (grouped: up to 4 right slices per MMA,
// see the kernel) and the stage's commits, from the one lane a single
// elect.sync picks. tm: TMEM base of the level accumulators (64 columns per
// level); ad / rd: shared-memory descriptors of left slice 0 / right slice 0
// of this stage (slice t is t * 4096 / 16 = 256 t descriptor units further,
// right slice u 128 u); idN: instruction descriptors for N = 64 N; acc0: 0 on
// the first k-tile (levels overwritten by the t = 0 MMAs); ebar / cbar /
// fbar: shared::cluster addresses of the stage's empty barrier, the cluster
// leader's (0: none) and tmem_full (0: not the last k-tile).
#define XB_MMA "@pe tcgen05.mma.cta_group::1.kind::i8 "
#define XB_COMMIT_TAIL                                                                        \
  "@pe tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n"          \
  "setp.ne.and.b32 pc, %9, 0, pe;\n"                                                          \
  "@pc tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n"          \
  "setp.ne.and.b32 pf, %10, 0, pe;\n"                                                         \
  "@pf tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n"         \
  "}\n"
#define XB_ISSUE_ARGS                                                                         \
  ::"r"(tm), "l"(ad), "l"(rd), "r"(id1), "r"(id2), "r"(id3), "r"(id4), "r"(acc0), "r"(ebar),  \
      "r"(cbar), "r"(fbar)                                                                    \
      : "memory"
#define XB_ISSUE_HEAD                                                                         \
  "{\n"                                                                                       \
  ".reg .pred pe, p0, pt, pc, pf;\n"                                                          \
  ".reg .b64 a1, a2, a3, a4, a5, a6, b4;\n"                                                   \
  ".reg .b32 d1, d2, d3, d4, d5, d6;\n"                                                       \
  "elect.sync _|pe, 0xffffffff;\n"                                                            \
  "setp.ne.b32 p0, %7, 0;\n"                                                                  \
  "setp.eq.b32 pt, %7, %7;\n"                                                                 \
  "add.u64 a1, %1, 256;\n"                                                                    \
  "add.u64 a2, %1, 512;\n"                                                                    \
  "add.u64 a3, %1, 768;\n"                                                                    \
  "add.u64 a4, %1, 1024;\n"                                                                   \
  "add.u64 a5, %1, 1280;\n"                                                                   \
  "add.u64 a6, %1, 1536;\n"                                                                   \
  "add.u64 b4, %2, 512;\n"                                                                    \
  "add.u32 d1, %0, 64;\n"                                                                     \
  "add.u32 d2, %0, 128;\n"                                                                    \
  "add.u32 d3, %0, 192;\n"                                                                    \
  "add.u32 d4, %0, 256;\n"                                                                    \
  "add.u32 d5, %0, 320;\n"                                                                    \
  "add.u32 d6, %0, 384;\n"

template <int S>
__device__ __forceinline__ void issue_tile(uint32_t tm, uint64_t ad, uint64_t rd, uint32_t id1,
                                           uint32_t id2, uint32_t id3, uint32_t id4,
                                           uint32_t acc0, uint32_t ebar, uint32_t cbar,
                                           uint32_t fbar) {
  static_assert(S == 4 || S == 6 || S == 7, "grouped issue lists exist for S = 4, 6, 7");
  if constexpr (S == 6) {
    // (t, u0, slices): (0,0,4) (0,4,2) (1,0,4) (1,4,1) (2,0,4) (3,0,3) (4,0,2) (5,0,1)
    // natural order (t outer). Measured alternatives, per cfg2 product: sorted
    // by N (every consecutive pair overlaps in its level range) 1.913 ms,
    // fewest overlapping transitions (B A G D C H E F) 1.865 ms, this 1.856 ms
    asm volatile(XB_ISSUE_HEAD
                 XB_MMA "[%0], %1, %2, %6, p0;\n"
                 XB_MMA "[d4], %1, b4, %4, p0;\n"
                 XB_MMA "[d1], a1, %2, %6, pt;\n"
                 XB_MMA "[d5], a1, b4, %3, pt;\n"
                 XB_MMA "[d2], a2, %2, %6, pt;\n"
                 XB_MMA "[d3], a3, %2, %5, pt;\n"
                 XB_MMA "[d4], a4, %2, %4, pt;\n"
                 XB_MMA "[d5], a5, %2, %3, pt;\n"
                 XB_COMMIT_TAIL XB_ISSUE_ARGS);
  } else if constexpr (S == 7) {
    // (0,0,4) (0,4,3) (1,0,4) (1,4,2) (2,0,4) (2,4,1) (3,0,4) (4,0,3) (5,0,2) (6,0,1)
    asm volatile(XB_ISSUE_HEAD
                 XB_MMA "[%0], %1, %2, %6, p0;\n"
                 XB_MMA "[d4], %1, b4, %5, p0;\n"
                 XB_MMA "[d1], a1, %2, %6, pt;\n"
                 XB_MMA "[d5], a1, b4, %4, pt;\n"
                 XB_MMA "[d2], a2, %2, %6, pt;\n"
                 XB_MMA "[d6], a2, b4, %3, pt;\n"
                 XB_MMA "[d3], a3, %2, %6, pt;\n"
                 XB_MMA "[d4], a4, %2, %5, pt;\n"
                 XB_MMA "[d5], a5, %2, %4, pt;\n"
                 XB_MMA "[d6], a6, %2, %3, pt;\n"
                 XB_COMMIT_TAIL XB_ISSUE_ARGS);
  } else {
    // S = 4: (0,0,4) (1,0,3) (2,0,2) (3,0,1)
    asm volatile(XB_ISSUE_HEAD
                 XB_MMA "[%0], %1, %2, %6, p0;\n"
                 XB_MMA "[d1], a1, %2, %5, pt;\n"
                 XB_MMA "[d2], a2, %2, %4, pt;\n"
                 XB_MMA "[d3], a3, %2, %3, pt;\n"
                 XB_COMMIT_TAIL XB_ISSUE_ARGS);
  }
}
#undef XB_MMA
#undef XB_COMMIT_TAIL
#undef XB_ISSUE_ARGS
#undef XB_ISSUE_HEAD

template <int S, int TC>
__global__ void __launch_bounds__(OTHREADS, 1)
    ozgemm_kernel(const int8_t* __restrict__ L, const int8_t* __restrict__ R, int64_t rows_p,
                  int64_t np, const int32_t* __restrict__ eL, const int32_t* __restrict__ eR,
                  int64_t M, int64_t N, int64_t K, double* __restrict__ C, int64_t ldc,
                  int64_t split_stride,
                  int64_t k_per_split, int accumulate, int tiles_n, int dbg, int cl) {
  using Cfg = OCfg<S>;
  static_assert(TC == 0 || S <= 6, "no TMEM A slots at S = 7");
  constexpr int NS = Cfg::NS;
  extern __shared__ unsigned char smem_raw_o[];
  unsigned char* smem = smem_raw_o + ((1024u - (su32(smem_raw_o) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* empty = full + NS;
  uint64_t* tmem_full = empty + NS;
  uint64_t* cempty = tmem_full + 1;  // [NS] cluster leader: stage free in all cl CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + NS);
  // cluster of cl CTAs = the n-tiles of one (m-tile, split): the leader
  // multicasts the left slices, which are then read from L2 once per m-tile
  const uint32_t crank = cl > 1 ? cluster_ctarank() : 0u;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (int)(blockIdx.x % tiles_n);
  const int64_t mt = blockIdx.x / tiles_n;
  const int64_t m0 = mt * OBM, n0 = (int64_t)nt * OBN;
  // dbg 64: Gram, only tiles on or above the diagonal are ever read;
  // dbg 128: the right operand is upper triangular (rows k >= n0 + OBN of
  // this n-tile are zero). Both come without clusters (cl = 1).
  if ((dbg & 64) && n0 + OBN - 1 < m0) return;
  const int64_t kbeg = (int64_t)blockIdx.y * k_per_split;
  int64_t kend = min(K, kbeg + k_per_split);
  if (dbg & 128) kend = min(kend, n0 + OBN);
  const int ktiles = kend > kbeg ? (int)((kend - kbeg + OBK - 1) / OBK) : 0;
  C += (int64_t)blockIdx.y * split_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
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
    // ---- producer: one bulk copy per operand per k-tile --------------------------
    if (lane == 0) {
      const int64_t kb0 = kbeg / OBK, lt = rows_p / OBM, rt = np / OBN;
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % NS;
        if (kt >= NS) {
          mbar_wait_park(&empty[s], ((kt / NS) & 1) ^ 1);
          if (cl > 1 && crank == 0) mbar_wait_park(&cempty[s], ((kt / NS) & 1) ^ 1);
        }
        unsigned char* st = smem + s * Cfg::STAGE;
        mbar_expect_tx(&full[s], Cfg::STAGE);
        const int8_t* lsrc = L + ((kb0 + kt) * lt + mt) * (S * Cfg::ATILE);
        if (cl == 1)
          bulk_load(st, lsrc, S * Cfg::ATILE, &full[s]);
        else if (crank == 0)
          bulk_load_mc(st, lsrc, S * Cfg::ATILE, &full[s], (uint16_t)((1u << cl) - 1));
        bulk_load(st + S * Cfg::ATILE, R + ((kb0 + kt) * rt + nt) * (S * Cfg::RTILE),
                  S * Cfg::RTILE, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA warp: tcgen05.cp of the left slices into a TMEM A slot, then
    // the S(S+1)/2 slice products (cp and mma run in issue order) -------------
    const uint32_t idesc = idesc_i8<S>();
    // instruction descriptors for N = 64, 128, 192, 256 (1-4 right slices)
    uint32_t idesc_n[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      idesc_n[i] = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(((i + 1) * OBN) >> 3) << 17);
    const bool grouped = !(dbg & 4);
    // left slices 0 .. TC-1 are staged in TMEM by tcgen05.cp; the rest feed
    // their MMAs from shared memory
    constexpr int tc = TC;
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
    const uint32_t cempty0 = cl > 1 ? mapa_rank(cempty, 0) : 0u;  // leader's cempty[0]
    const uint32_t sbase = su32(smem);
    constexpr bool kLean = TC == 0 && (S == 4 || S == 6 || S == 7);
    if (kLean && (dbg & ~(64 | 128)) == 0) {
      if constexpr (kLean) {
      // Production path: ONE elect per k-tile for the grouped MMAs and the
      // commits together (issue_tile), shared-memory descriptors advanced by
      // adds, the stage index and phase kept incrementally. The generic loop
      // below spends ~20 uniform-datapath instructions per MMA (elect, vote,
      // descriptor assembly, experiment branches): its issue time per k-tile
      // was ~60 % of the k-tile's tensor time and paced the kernel.
      const uint64_t ad0 = smem_desc(sbase, 256, 0, 128);
      const uint64_t rd0 = smem_desc(sbase + (uint32_t)(S * Cfg::ATILE), 256, 0, 128);
      constexpr uint64_t kStep = (uint64_t)(Cfg::STAGE >> 4);
      const uint32_t e0 = su32(&empty[0]), tf = su32(tmem_full);
      uint64_t ad = ad0, rd = rd0;
      uint32_t st = 0, ph = 0;
      for (int kt = 0; kt < ktiles; ++kt) {
        mbar_wait(&full[st], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        issue_tile<S>(tm, ad, rd, idesc_n[0], idesc_n[1], idesc_n[2], idesc_n[3],
                      kt > 0 ? 1u : 0u, e0 + 8u * st, cl > 1 ? cempty0 + 8u * st : 0u,
                      kt == ktiles - 1 ? tf : 0u);
        ad += kStep;
        rd += kStep;
        if (++st == NS) {
          st = 0;
          ph ^= 1;
          ad = ad0;
          rd = rd0;
        }
      }
      }
    } else
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % NS, a = kt & 1;
      mbar_wait(&full[s], (kt / NS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t aslot = tm + (uint32_t)(Cfg::ACC_COLS + a * Cfg::ASLOT);
      const uint32_t abase = sbase + (uint32_t)(s * Cfg::STAGE);
      const uint32_t rbase = abase + (uint32_t)(S * Cfg::ATILE);
      if (!(dbg & 1)) {
#pragma unroll
        for (int t = 0; t < S; ++t)
          if (t < tc)
            cp_128x256b(aslot + (uint32_t)(t * (OBK / 4)),
                        smem_desc(abase + t * Cfg::ATILE, 256, 0, 128));
      }
      const uint32_t first = kt > 0 ? 1u : 0u;
      // Grouped: the right slices u0..u0+3 sit back to back in shared memory
      // (one 256-row K-major operand) and the level accumulators back to
      // back in TMEM, so ONE N=256 MMA of A slice t writes the pairs
      // (t, u0..u0+3) into levels t+u0..t+u0+3 — 8 MMAs per k-tile instead
      // of S(S+1)/2 = 21 for S = 6 (XB_OZ_GROUPED=0: one MMA per pair).
#pragma unroll
      for (int t = 0; t < S; ++t) {
        if (dbg & 2) break;
        if (grouped) {
#pragma unroll
          for (int u0 = 0; u0 < S - t; u0 += 4) {
            const int nsl = (S - t - u0) < 4 ? (S - t - u0) : 4;
            if (t < tc)
              mma_i8(tm + (uint32_t)((t + u0) * OBN), aslot + (uint32_t)(t * (OBK / 4)),
                     smem_desc(rbase + u0 * Cfg::RTILE, 256, 0, 128), idesc_n[nsl - 1],
                     t > 0 ? 1u : first);
            else
              mma_i8_ss(tm + (uint32_t)((t + u0) * OBN),
                        smem_desc(abase + t * Cfg::ATILE, 256, 0, 128),
                        smem_desc(rbase + u0 * Cfg::RTILE, 256, 0, 128), idesc_n[nsl - 1],
                        t > 0 ? 1u : first);
          }
        } else {
#pragma unroll
          for (int u = 0; u < S - t; ++u) {
            const int d = t + u;  // level (t + 1) + (u + 1) - 2
            mma_i8(tm + (uint32_t)(d * OBN), aslot + (uint32_t)(t * (OBK / 4)),
                   smem_desc(rbase + u * Cfg::RTILE, 256, 0, 128), idesc, t > 0 ? 1u : first);
          }
        }
      }
      // (measured: issuing this block from one elected lane, as ozf_kernel
      // does, is slower here: 2.14 -> 2.33 ms per cfg2 product)
      commit_elect(&empty[s]);
      if (cl > 1) commit_elect_cluster(cempty0 + (uint32_t)(s * sizeof(uint64_t)));
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
  if (cl > 1)
    cluster_sync_all();  // no CTA leaves while a peer may still multicast / arrive
  else
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
  constexpr unsigned long long kBias = 0x80808080808080ULL >> (8 * (8 - S));  // S - 1 digits
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
// A range up to 256x wider (kOzRange7) takes one more digit slice (S = 7: 55
// bits, 28 slice pairs instead of 21) instead of the 3.7x slower DMMA path:
// *wide = 1. Beyond that *wide = 2 (DMMA).
constexpr double kOzRange = 64.0;
constexpr double kOzRange7 = 64.0 * 256.0;
__device__ __forceinline__ void range_vote(int* wide, double m, double mean_sq) {
  if (!(mean_sq <= DBL_MAX) || m * m > kOzRange7 * kOzRange7 * mean_sq) atomicMax(wide, 2);
  else if (m * m > kOzRange * kOzRange * mean_sq) atomicMax(wide, 1);
}

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
    if (wide) range_vote(wide, m, ss / (double)cols);
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
  if (wide && css) range_vote(wide, m, css[c] / (double)rows);
}

// Row AND column max |x| / sum of squares of A in ONE pass (the slicing
// pass needs both exponent sets before it starts). Block tile 512 rows x 256
// columns: each warp reads 2 KB of a row per step (8 coalesced 256-byte
// loads), reduces the row partial by shuffle, and keeps
// 8 column partials per lane that the block combines in shared memory.
// Partials go to scratch without atomics — per (row, column tile) and per
// (row tile, column) — and two small kernels finish them in a fixed order.
constexpr int RC_ROWS = 512, RC_COLS = 256;

// Row AND column max |x| / sum of squares of A in ONE pass. Block tile =
// 512 rows x 256 columns: each warp reads 256 columns of a row per step —
// 8 coalesced 8-byte loads per lane for double; for float 2 16-byte loads
// per lane and 2 rows in flight — reduces the row partial by shuffle, and
// keeps 8 column partials per lane that the block combines in shared
// memory. Partials go to scratch without atomics — per (row, column tile)
// and per (row tile, column) — and two small kernels finish them in a
// fixed order.
template <typename T>
__device__ __forceinline__ int rc_col(int tx, int j) {
  // the column (within the tile) of a lane's j-th value
  if constexpr (sizeof(T) == 4)
    return 4 * tx + (j & 3) + 128 * (j >> 2);
  else
    return tx + 32 * j;
}

template <typename T>
__global__ void __launch_bounds__(256, 4)
    rc_stats_kernel(const T* __restrict__ X, int64_t rows, int64_t cols, int64_t ldx,
                    double2* __restrict__ rpart, double2* __restrict__ cpart) {
  constexpr bool F = sizeof(T) == 4;
  constexpr int U = F ? 2 : 1;  // rows in flight per warp
  __shared__ double sm[8][RC_COLS + 1], sq[8][RC_COLS + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t ct = blockIdx.x, rt = blockIdx.y;
  const int64_t nct = gridDim.x;
  const int64_t c0 = ct * RC_COLS, r0 = rt * RC_ROWS;
  const int64_t rend = min(rows, r0 + RC_ROWS);
  // float rows are 16-byte loaded when the whole tile row is in range and aligned
  const bool vec = F && c0 + RC_COLS <= cols && (ldx % 4) == 0 &&
                   (reinterpret_cast<uintptr_t>(X) % 16) == 0;
  double cm[8], cs[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) cm[j] = cs[j] = 0.0;
  bool colok[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) colok[j] = c0 + rc_col<T>(tx, j) < cols;
  for (int64_t rb = r0 + ty; rb < rend; rb += 8 * U) {
    T v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = rb + 8 * u;
      const T* xr = X + r * ldx + c0;
      if constexpr (F) {
        if (vec) {
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
          if (r < rend) {
            a = __ldcs(reinterpret_cast<const float4*>(xr) + tx);
            b = __ldcs(reinterpret_cast<const float4*>(xr + 128) + tx);
          }
          v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w;
          v[u][4] = b.x; v[u][5] = b.y; v[u][6] = b.z; v[u][7] = b.w;
          continue;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int cc = rc_col<T>(tx, j);
        v[u][j] = (r < rend && colok[j]) ? __ldcs(xr + cc) : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double m = 0.0, ss = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double x = (double)v[u][j], a = fabs(x);
        m = fmax(m, a);
        ss = fma(x, x, ss);
        cm[j] = fmax(cm[j], a);
        cs[j] = fma(x, x, cs[j]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
      }
      const int64_t r = rb + 8 * u;
      if (tx == 0 && r < rend) rpart[r * nct + ct] = make_double2(m, ss);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sm[ty][rc_col<T>(tx, j)] = cm[j];
    sq[ty][rc_col<T>(tx, j)] = cs[j];
  }
  __syncthreads();
  const int64_t c = c0 + threadIdx.x;
  if (c < cols) {
    double m = 0.0, ss = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      m = fmax(m, sm[w][threadIdx.x]);
      ss += sq[w][threadIdx.x];
    }
    cpart[rt * cols + c] = make_double2(m, ss);
  }
}

// Fast path, float A (the f32 configs' 64 GB pass): the same partials with float
// arithmetic — the generic kernel's f32 -> f64 conversion and f64 max / fma
// per element made it issue-bound at ~3 TB/s (ncu: 79 % issue slots busy,
// DRAM 36 %). max |x| is exact in float; the sums of squares are float per
// lane and row (256 terms) and per column and tile (512 terms), which is
// plenty for a range guard, and an overflowing one reads as "wide" (DMMA),
// never as a false "narrow". Each warp takes 8 rows per step (16 loads of
// 16 bytes in flight per lane) and reduces the 8 row partials across lanes
// by halving exchanges (9 shuffles per quantity instead of 40). Double A
// takes the same kernel with f64 arithmetic and 4 rows per step (32 loads
// of 8 bytes in flight per lane; the generic kernel kept 8).
template <typename T>
__device__ __forceinline__ T rc_absmax(T a, T b) {
  if constexpr (sizeof(T) == 4)
    return fmaxf(a, b);
  else
    return fmax(a, b);
}

template <typename T>
__global__ void __launch_bounds__(256, 2)
    rc_stats_fast_kernel(const T* __restrict__ X, int64_t rows, int64_t cols, int64_t ldx,
                         double2* __restrict__ rpart, double2* __restrict__ cpart) {
  constexpr bool F = sizeof(T) == 4;
  constexpr int RR = F ? 8 : 4;  // rows per warp step
  __shared__ T sm[8][RC_COLS + 1], sq[8][RC_COLS + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t ct = blockIdx.x, rt = blockIdx.y;
  const int64_t nct = gridDim.x;
  const int64_t c0 = ct * RC_COLS, r0 = rt * RC_ROWS;
  const int64_t rend = min(rows, r0 + RC_ROWS);
  const bool full_cols = c0 + RC_COLS <= cols;
  T cm[8], cs[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) cm[j] = cs[j] = T(0);
  for (int64_t rb = r0 + RR * ty; rb < rend; rb += 8 * RR) {
    T v[RR][8];
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      const int64_t r = rb + i;
      const T* xr = X + r * ldx + c0;
      if constexpr (F) {
        if (full_cols) {
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
          if (r < rend) {
            a = __ldcs(reinterpret_cast<const float4*>(xr) + tx);
            b = __ldcs(reinterpret_cast<const float4*>(xr + 128) + tx);
          }
          v[i][0] = a.x; v[i][1] = a.y; v[i][2] = a.z; v[i][3] = a.w;
          v[i][4] = b.x; v[i][5] = b.y; v[i][6] = b.z; v[i][7] = b.w;
          continue;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int cc = rc_col<T>(tx, j);
        v[i][j] = (r < rend && (full_cols || c0 + cc < cols)) ? __ldcs(xr + cc) : T(0);
      }
    }
    T rm[RR], rs[RR];
#pragma unroll
    for (int i = 0; i < RR; ++i) {
      rm[i] = T(0);
      rs[i] = T(0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const T x = v[i][j], a = x < T(0) ? -x : x;
        rm[i] = rc_absmax(rm[i], a);
        rs[i] = fma(x, x, rs[i]);
        cm[j] = rc_absmax(cm[j], a);
        cs[j] = fma(x, x, cs[j]);
      }
    }
    // halving exchanges: at offset o a lane keeps the upper or lower half of
    // its remaining rows (by lane bit o) and takes the partner's partials of
    // that half; once one row is left the remaining offsets reduce it fully
    int ri = 0;
#pragma unroll
    for (int n = RR, o = 16; o > 0; o >>= 1) {
      if (n > 1) {
        const bool hi = tx & o;
#pragma unroll
        for (int k = 0; k < n / 2; ++k) {
          const T sendm = hi ? rm[k] : rm[k + n / 2], sends = hi ? rs[k] : rs[k + n / 2];
          const T gm = __shfl_xor_sync(0xffffffffu, sendm, o);
          const T gs = __shfl_xor_sync(0xffffffffu, sends, o);
          rm[k] = rc_absmax(hi ? rm[k + n / 2] : rm[k], gm);
          rs[k] = (hi ? rs[k + n / 2] : rs[k]) + gs;
        }
        if (hi) ri += n / 2;
        n /= 2;
      } else {
        rm[0] = rc_absmax(rm[0], __shfl_xor_sync(0xffffffffu, rm[0], o));
        rs[0] += __shfl_xor_sync(0xffffffffu, rs[0], o);
      }
    }
    const int64_t r = rb + ri;
    if ((tx & (32 / RR - 1)) == 0 && r < rend)
      rpart[r * nct + ct] = make_double2((double)rm[0], (double)rs[0]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sm[ty][rc_col<T>(tx, j)] = cm[j];
    sq[ty][rc_col<T>(tx, j)] = cs[j];
  }
  __syncthreads();
  const int64_t c = c0 + threadIdx.x;
  if (c < cols) {
    double m = 0.0, ss = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      m = fmax(m, (double)sm[w][threadIdx.x]);
      ss += (double)sq[w][threadIdx.x];
    }
    cpart[rt * cols + c] = make_double2(m, ss);
  }
}

// e[i] from the partials part[i * stride + t * tstep], t < parts; `len` =
// elements per row/column (the range guard's mean square)
__global__ void rc_finish_kernel(const double2* __restrict__ part, int64_t count, int64_t parts,
                                 int64_t stride, int64_t tstep, int64_t len,
                                 int32_t* __restrict__ e, int* __restrict__ wide) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double m = 0.0, ss = 0.0;
  for (int64_t t = 0; t < parts; ++t) {
    const double2 p = part[i * stride + t * tstep];
    m = fmax(m, p.x);
    ss += p.y;
  }
  e[i] = slice_exp(m);
  // (a non-finite sum of squares — float partials that overflowed — counts
  // as wide)
  if (wide) range_vote(wide, m, ss / (double)len);
}

template <int S>
__device__ __forceinline__ void slice7(double x, int e, int8_t* out, int64_t plane) {
  int a[S];
  slice_digits<S>(x, e, a);
#pragma unroll
  for (int t = 0; t < S; ++t) out[t * plane] = (int8_t)a[t];
}

// Slices of a left operand straight from A, in one pass over A (one read):
// PR = the row-scaled slices of A (rows of A, K = columns; for Y = A X) and
// PC = the column-scaled slices of A^T (columns of A, K = rows; for
// Z = A^T Q), both in the interleaved tile layout (il_off<128>). Either may be
// null. Block tile = 128 rows x 32 columns of A (32 KB in shared memory):
// that is exactly one 4 KB interleaved tile per slice of PR, and four 1 KB
// contiguous runs per slice of PC, so every warp store is a contiguous
// 128-byte run (thread t writes the t-th 4-byte word of the run).
template <int S>
__global__ void __launch_bounds__(256)
    slice_both_kernel(const double* __restrict__ X, int64_t m, int64_t n, int64_t ldx,
                      const int32_t* __restrict__ er, const int32_t* __restrict__ ec,
                      int8_t* __restrict__ PR, int64_t mp, int64_t kpn, int8_t* __restrict__ PC,
                      int64_t np, int64_t kpm) {
  __shared__ double tile[128][33];
  __shared__ int ser[128], sec[32];
  const int64_t r0 = (int64_t)blockIdx.x * 128, c0 = (int64_t)blockIdx.y * 32;
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  {
    // all 16 loads of a thread in flight before the shared-memory stores (a
    // load -> store loop left one load in flight: 58 % of DRAM bandwidth)
    double v[16];
    const int64_t c = c0 + tx;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int64_t r = r0 + ty + 8 * k;
      v[k] = (r < m && c < n) ? __ldcs(X + r * ldx + c) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[ty + 8 * k][tx] = v[k];
  }
  if (t < 128) ser[t] = (er && r0 + t < m) ? er[r0 + t] : 0;
  if (t < 32) sec[t] = (ec && c0 + t < n) ? ec[c0 + t] : 0;
  __syncthreads();
  if (PR && c0 < kpn) {
    // the (k-block c0/32, row tile r0/128) interleaved tile, word by word
    int8_t* base = PR + ((c0 >> 5) * (mp / 128) + (r0 >> 7)) * (int64_t)(S * 4096);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int w = t + 256 * u;
      const int rr = ((w >> 6) << 3) | ((w >> 2) & 7);
      const int kk = ((w >> 5) & 1) * 16 + (w & 3) * 4;
      uint32_t word[S];
#pragma unroll
      for (int q = 0; q < S; ++q) word[q] = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int d[S];
        slice_digits<S>(tile[rr][kk + j], ser[rr], d);
#pragma unroll
        for (int q = 0; q < S; ++q) word[q] |= (uint32_t)(uint8_t)(int8_t)d[q] << (8 * j);
      }
#pragma unroll
      for (int q = 0; q < S; ++q) reinterpret_cast<uint32_t*>(base + q * 4096)[w] = word[q];
    }
  }
  if (PC && c0 < np) {
    // rows c0..c0+31 of A^T (a 32-row slab of row tile c0/128), k-blocks r0/32 + kb
    const int rr0 = (int)(c0 & 127);
    const int cc = ((t >> 6) << 3) | ((t >> 2) & 7);  // 0..31: row within the slab
    const int kk = ((t >> 5) & 1) * 16 + (t & 3) * 4;
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const int64_t kblk = (r0 >> 5) + kb;
      if (kblk * 32 >= kpm) break;
      int8_t* base = PC + (kblk * (np / 128) + (c0 >> 7)) * (int64_t)(S * 4096) + (rr0 >> 3) * 256;
      uint32_t word[S];
#pragma unroll
      for (int q = 0; q < S; ++q) word[q] = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int d[S];
        slice_digits<S>(tile[kb * 32 + kk + j][cc], sec[cc], d);
#pragma unroll
        for (int q = 0; q < S; ++q) word[q] |= (uint32_t)(uint8_t)(int8_t)d[q] << (8 * j);
      }
#pragma unroll
      for (int q = 0; q < S; ++q) reinterpret_cast<uint32_t*>(base + q * 4096)[t] = word[q];
    }
  }
}

// Right operand: X (K x N, ldx) -> column-scaled slices of X^T in the
// interleaved layout of 64-row tiles (il_off<64>), zero padded to (np, kp).
template <int S, int TR>
__global__ void __launch_bounds__(256)
    slice_right_kernel(const double* __restrict__ X, int64_t K, int64_t N, int64_t ldx,
                       const int32_t* __restrict__ e, int8_t* __restrict__ P, int64_t np,
                       int64_t kp) {
  __shared__ double tile[32][33];
  __shared__ int se[32];
  const int64_t k0 = (int64_t)blockIdx.x * 32, n0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y, t = ty * 32 + tx;
  for (int i = ty; i < 32; i += 8) {
    const int64_t k = k0 + i, c = n0 + tx;
    tile[i][tx] = (k < K && c < N) ? X[k * ldx + c] : 0.0;
  }
  if (ty == 0) se[tx] = (n0 + tx < N) ? e[n0 + tx] : 0;
  __syncthreads();
  const int a = t >> 3, b4 = (t & 7) * 4;
  if (n0 + a < np && k0 < kp) {
    uint32_t w[S];
#pragma unroll
    for (int q = 0; q < S; ++q) w[q] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int d[S];
      slice_digits<S>(tile[b4 + j][a], se[a], d);
#pragma unroll
      for (int q = 0; q < S; ++q) w[q] |= (uint32_t)(uint8_t)(int8_t)d[q] << (8 * j);
    }
#pragma unroll
    for (int q = 0; q < S; ++q)
      *reinterpret_cast<uint32_t*>(P + il_off<TR>(n0 + a, k0 + b4, q, S, np)) = w[q];
  }
}

template <int S>
void launch_oz(const int8_t* L, const int8_t* R, int64_t rows_p, int64_t np, const int32_t* eL,
               const int32_t* eR, int64_t M, int64_t N, int64_t K, double* out, int64_t ldo,
               int64_t stride, int64_t kps, int splits, int acc, int tri, cudaStream_t st) {
  using Cfg = OCfg<S>;
  // Left slices straight from shared memory (TC = 0) by default. Staging
  // them in TMEM with tcgen05.cp (XB_OZ_TC=S) saves shared-memory reads for
  // the slices two MMAs use, but the copies execute in order with the MMAs
  // on the tensor pipe: cfg2 product 2.14 ms at 66 % tensor-active staged
  // (2 staged: 1.92 ms) vs 1.90 ms at 84 % unstaged.
  static const bool staged = [] {
    const char* e = knob("XB_OZ_TC");
    return e && atoi(e) == S;
  }();
  auto kern = ozgemm_kernel<S, 0>;
  if constexpr (S <= 6) {
    if (staged) kern = ozgemm_kernel<S, S>;
  }
  XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int64_t tn = ceil_div(N, OBN), tm = ceil_div(M, OBM);
  XB_REQUIRE(tn * tm < ((int64_t)1 << 31) && splits < 65536, XB_EUNSUPPORTED,
             "ozgemm: grid too large");
  dim3 grid((unsigned)(tn * tm), (unsigned)splits);
  static const int dbg = [] {
    const char* e = knob("XB_OZ_DBG");
    const char* g = knob("XB_OZ_GROUPED");
    return (e ? atoi(e) : 0) | ((g && atoi(g) == 0) ? 4 : 0);
  }();
  // the n-tiles of an (m-tile, split) share the left slices by multicast
  // (XB_OZ_CLUSTER=0 disables)
  static const bool cluster_on = [] {
    const char* e = knob("XB_OZ_CLUSTER");
    return !(e && atoi(e) == 0);
  }();
  const int cl = (cluster_on && tri == 0 && tn >= 2 && tn <= 4) ? (int)tn : 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(OTHREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  XB_CUDA(cudaLaunchKernelEx(&cfg, kern, L, R, rows_p, np, eL, eR, M, N, K, out, ldo, stride,
                             kps, acc, (int)tn,
                             dbg | (tri == 1 ? 64 : 0) | (tri == 2 ? 128 : 0), cl));
  check_launch("ozgemm");
}

// ---- float32 A on the int8 pipe: slices made on the fly ---------------------
//
// The f32 configs' products (Y = A X, Z = A^T Q with A in float32) with A
// sliced into FS = 3 int8 digits (22 bits relative to its row / column
// scale, round to nearest) INSIDE the GEMM: the raw f32 A
// tile arrives by TMA exactly as in tgemm.cu, converter warps turn each
// row's 32 values into 3 packed digit planes and store them into a TMEM A
// slot (tcgen05.st), and the MMA warp issues the 6 pairs (t, u), t + u < 3,
// of tcgen05.mma.kind::i8 (M=128, N=BN, K=32) against the right slices
// (the sketch X, sliced per product) into three int32 level accumulators.
// int32 sums are exact, so no mid-chain draining is needed (K per split
// <= 32768); the epilogue weights the levels in f64. The products are as
// accurate as an f32 SGEMM or better, at half the tensor work of 3xTF32
// (6 int8 products = 1.5 tf32-product equivalents per useful flop) and
// far less energy per flop.
constexpr int FS = 3;
constexpr int FBM = 128, FBK = 32;
constexpr int FEPI = 4;                      // epilogue warps
// converter warps: FPH k-tile phases x 4 TMEM lane quadrants; the warps of
// phase h convert the whole 128 x 32 tile of every k-tile kt = h (mod FPH),
// so each warp has FPH MMA k-tiles of time per tile it converts and its
// fixed per-tile costs (barrier waits, TMEM store wait, arrive) are paid once
// per 32 k values instead of once per 8
constexpr int FPH = 3;
constexpr int FCONV = 4 * FPH;
constexpr int FTHREADS = 32 * (2 + FCONV + FEPI);  // producer, MMA, converters, epilogue

// One stage ring: raw A tile + the right slices of a k-tile per stage.
// (Measured: separate A and R rings, the A stage released by the converters
// and each ring refilled by its own thread, were no faster for TN and much
// slower for the clustered NN launch.)
template <int BN>
struct FCfg {
  static constexpr int A_BYTES = FBM * FBK * 4;            // raw f32 A tile (TMA)
  static constexpr int R_BYTES = FS * BN * FBK;            // FS right slices, BN rows x 32 B
  static constexpr int STAGE = ((A_BYTES + R_BYTES + 1023) / 1024) * 1024;
  // the stage count is a multiple of FPH: every k-tile that uses a given
  // stage belongs to the same converter phase, so each converter warp meets
  // that stage's barrier phases in order
  static constexpr int NS0 = (200 * 1024) / STAGE > 6 ? 6 : (200 * 1024) / STAGE;
  static constexpr int NS = NS0 - NS0 % FPH;
  static constexpr int BAR_OFF = NS * STAGE;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;
  static constexpr int ACC_COLS = FS * BN;
  static constexpr int ASLOT = FS * (FBK / 4);             // 24 TMEM columns
  // A slots (converters run NA k-tiles ahead of the MMAs): what TMEM leaves,
  // a multiple of FPH for the same reason as NSA
  static constexpr int NA0 = (512 - ACC_COLS) / ASLOT > 6 ? 6 : (512 - ACC_COLS) / ASLOT;
  static constexpr int NA = NA0 - NA0 % FPH;
  static_assert(NA >= FPH && NS >= FPH, "slot / stage counts");
  static_assert(ACC_COLS + NA * ASLOT <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

template <int BN>
__device__ __forceinline__ uint32_t idesc_i8n() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(FBM >> 4) << 24);
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

template <int BN, bool TRANS_A>
__global__ void __launch_bounds__(FTHREADS, 1)
    ozf_kernel(const __grid_constant__ CUtensorMap tmA, const int8_t* __restrict__ R, int64_t np,
               const int32_t* __restrict__ eL, const int32_t* __restrict__ eR, int64_t M,
               int64_t N, int64_t K, double* __restrict__ C, int64_t ldc, int64_t split_stride,
               int64_t k_per_split, int accumulate, int tiles_n, int tiles_m, int splits,
               int group_m, int cl_dbg) {
  using Cfg = FCfg<BN>;
  constexpr int NS = Cfg::NS, NA = Cfg::NA;
  // low byte: cluster size; above: XB_OZF_DBG timing experiments (results
  // are wrong with any bit set): 1 converters skip the A tile, 2 only the
  // t = 0 MMAs, 4 no A tile load (with 1), 16 no right-slice load
  const int cl = cl_dbg & 0xff, dbg = cl_dbg >> 8;
  extern __shared__ unsigned char smem_raw_f[];
  unsigned char* smem = smem_raw_f + ((1024u - (su32(smem_raw_f) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* conv = full + NS;     // count 4: the converter warps of the stage's phase
  uint64_t* empty = conv + NS;    // MMA commit: stage (and the A slot of k-tile kt) free
  uint64_t* cempty = empty + NS;  // cluster leader: stage free in all cl CTAs
  uint64_t* tmem_full = cempty + NS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  // cluster = the n-tiles of one (m-tile, split); the leader multicasts the
  // raw A tile (read once per m-tile instead of once per n-tile)
  const uint32_t crank = cl > 1 ? cluster_ctarank() : 0u;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // raster as tgemm.cu: n fastest, m within groups of group_m, then splits
  int64_t Lb = blockIdx.x;
  const int nt = (int)(Lb % tiles_n);
  Lb /= tiles_n;
  const int64_t per_group = (int64_t)group_m * splits;
  const int64_t mg = Lb / per_group;
  const int64_t w = Lb - mg * per_group;
  const int gsz = (int)min((int64_t)group_m, (int64_t)tiles_m - mg * group_m);
  const int split = (int)(w / gsz);
  const int64_t mt = mg * group_m + (w - (int64_t)split * gsz);
  const int64_t m0 = mt * FBM, n0 = (int64_t)nt * BN;
  const int64_t kbeg = (int64_t)split * k_per_split;
  const int64_t kend = min(K, kbeg + k_per_split);
  const int ktiles = kend > kbeg ? (int)((kend - kbeg + FBK - 1) / FBK) : 0;
  C += (int64_t)split * split_stride;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
      mbar_init(&cempty[s], cl);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (cl > 1)
    cluster_sync_all();
  else
    __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- producer: raw A tile (TMA; the cluster leader multicasts) + the
    // right slices (one bulk copy) ---------------------------------------------
    if (lane == 0) {
      const int64_t kb0 = kbeg / FBK, rt = np / BN;
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % NS;
        if (kt >= NS) {
          mbar_wait_park(&empty[s], ((kt / NS) & 1) ^ 1);
          if (cl > 1 && crank == 0) mbar_wait_park(&cempty[s], ((kt / NS) & 1) ^ 1);
        }
        unsigned char* st = smem + s * Cfg::STAGE;
        const int32_t k0 = (int32_t)(kbeg + (int64_t)kt * FBK);
        mbar_expect_tx(&full[s], ((dbg & 4) ? 0 : Cfg::A_BYTES) + ((dbg & 16) ? 0 : Cfg::R_BYTES));
        // TRANS_A: [BK][BM], M inner; else [BM][BK], 128B swizzle
        const int32_t ca = TRANS_A ? (int32_t)m0 : k0, cb = TRANS_A ? k0 : (int32_t)m0;
        if (dbg & 4) {
        } else if (cl == 1)
          tma_load_2d(st, &tmA, &full[s], ca, cb);
        else if (crank == 0)
          tma_load_2d_mc(st, &tmA, &full[s], ca, cb, (uint16_t)((1u << cl) - 1));
        if (!(dbg & 16))
          bulk_load(st + Cfg::A_BYTES, R + ((kb0 + kt) * rt + nt) * (int64_t)Cfg::R_BYTES,
                    Cfg::R_BYTES, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ---- MMA: A digit planes from TMEM, right slices from shared memory ------
    // (issued by one elected lane per k-tile: per-instruction elect / vote /
    // uniformise sequences otherwise dominate this warp's loop)
    const uint32_t idesc = idesc_i8n<BN>();
    const uint32_t cempty0 = cl > 1 ? mapa_rank(cempty, 0) : 0u;
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % NS, a = kt % NA;
      mbar_wait(&conv[s], (kt / NS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t aslot = tmem + (uint32_t)(Cfg::ACC_COLS + a * Cfg::ASLOT);
      const uint32_t rbase = su32(smem + s * Cfg::STAGE + Cfg::A_BYTES);
      const uint32_t first = kt > 0 ? 1u : 0u;
      if (elect_one()) {
        // grouped as in ozgemm_kernel: G = 256 / BN consecutive right slices
        // per MMA land in consecutive level accumulators
        constexpr int G = 256 / BN;
#pragma unroll
        for (int t = 0; t < ((dbg & 2) ? 1 : FS); ++t)
#pragma unroll
          for (int u0 = 0; u0 < FS - t; u0 += G) {
            const int nsl = (FS - t - u0) < G ? (FS - t - u0) : G;
            const uint32_t id = (idesc & ~(0x3Fu << 17)) | ((uint32_t)((nsl * BN) >> 3) << 17);
            mma_i8_1(tmem + (uint32_t)((t + u0) * BN), aslot + (uint32_t)(t * (FBK / 4)),
                     smem_desc(rbase + u0 * BN * FBK, 256, 0, 128), id, t > 0 ? 1u : first);
          }
        commit_1(su32(&empty[s]));
        if (cl > 1) commit_1(cempty0 + (uint32_t)(s * sizeof(uint64_t)));
        if (kt == ktiles - 1) commit_1(su32(tmem_full));
      }
      __syncwarp();
    }
  } else if (warp < 2 + FCONV) {
    // ---- converters: row m's 32 f32 values of k-tile kt -> 3 packed digit
    // planes in TMEM. v = rint(x 2^(22 - e)), |v| < 2^22 (7 + 8 + 7
    // bits), comes out of ONE fma: x 2^(22-e) + 1.5 2^23 has ulp 1, so its bit
    // pattern minus the constant's is v, rounded to nearest even (no F2I).
    // u = v + 0x8080 makes the two lower balanced digits plain bytes with
    // the top bit flipped (w = u ^ 0x8080 restores them); byte 2 of w is the
    // top digit. Byte permutes gather 4 elements' digits per TMEM word.
    const int m = 32 * (warp & 3) + lane;  // TMEM lane quadrant = warp id % 4
    const int h = (warp - 2) >> 2;         // k-tile phase
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const int e = (m0 + m < M) ? eL[m0 + m] : 0;
    const float sc = __int_as_float((127 + min(127, max(-126, 22 - e))) << 23);  // 2^(22-e)
    constexpr float kMagic = 12582912.0f;                       // 1.5 2^23
    const int kOff = __float_as_int(kMagic) - 0x8080;
    for (int kt = h; kt < ktiles; kt += FPH) {
      const int s = kt % NS, a = kt % NA;
      mbar_wait_park(&full[s], (kt / NS) & 1);
      const unsigned char* raw = smem + s * Cfg::STAGE;
      uint32_t wd[FS][8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // 16-byte chunk c = k 4c .. 4c+3
        float4 v;
        if (dbg & 1) {
          v = make_float4(1.f, 2.f, 3.f, (float)c);
        } else if constexpr (!TRANS_A) {
          v = *reinterpret_cast<const float4*>(raw + m * 128 + ((c ^ (m & 7)) << 4));
        } else {
          const float* rf = reinterpret_cast<const float*>(raw);
          v.x = rf[(4 * c + 0) * FBM + m];
          v.y = rf[(4 * c + 1) * FBM + m];
          v.z = rf[(4 * c + 2) * FBM + m];
          v.w = rf[(4 * c + 3) * FBM + m];
        }
        // (the 0x80 flips of the two lower digits are applied to the packed
        // words: one xor per 4 elements and digit)
        const uint32_t w0 = (uint32_t)(__float_as_int(fmaf(v.x, sc, kMagic)) - kOff);
        const uint32_t w1 = (uint32_t)(__float_as_int(fmaf(v.y, sc, kMagic)) - kOff);
        const uint32_t w2 = (uint32_t)(__float_as_int(fmaf(v.z, sc, kMagic)) - kOff);
        const uint32_t w3 = (uint32_t)(__float_as_int(fmaf(v.w, sc, kMagic)) - kOff);
        const uint32_t lo = __byte_perm(w0, w1, 0x5140), hi = __byte_perm(w2, w3, 0x5140);
        wd[2][c] = __byte_perm(lo, hi, 0x5410) ^ 0x80808080u;  // byte 0: lowest digit
        wd[1][c] = __byte_perm(lo, hi, 0x7632) ^ 0x80808080u;  // byte 1
        wd[0][c] = __byte_perm(__byte_perm(w0, w1, 0x62), __byte_perm(w2, w3, 0x62), 0x5410);
      }
      // the slot wait comes after the loads and digit arithmetic, so only the
      // TMEM stores sit between an MMA group's completion and the next arrive.
      // Slot a is free once the MMAs of k-tile kt - NA completed: the commit
      // that frees that k-tile's stage says exactly that (NS and NA are
      // multiples of FPH, so this warp meets the barrier's phases in order)
      if (kt >= NA) {
        const int kp = kt - NA;
        mbar_wait_park(&empty[kp % NS], (kp / NS) & 1);
      }
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t tbase = tmem + lane_base + (uint32_t)(Cfg::ACC_COLS + a * Cfg::ASLOT);
#pragma unroll
      for (int t = 0; t < FS; ++t) tmem_st8(tbase + (uint32_t)(t * (FBK / 4)), wd[t]);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
  } else {
    // ---- epilogue: levels -> f64, * 2^-(14+8d), sum, * 2^(e_i + f_j) ---------
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
    for (int c0 = 0; c0 < BN; c0 += 16) {
      double acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0;
      if (ktiles > 0) {
#pragma unroll 1
        for (int d = 0; d < FS; ++d) {
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
              "%11, %12, %13, %14, %15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tmem + lane_base + (uint32_t)(d * BN + c0)));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          // A digits carry 22 bits (x 2^(e-22)), the right slices 23 (x 2^(f-23)):
          // level d = t + u weighs 2^(e + f) 2^-(13 + 8 d)
          const double sc = ldexp(1.0, -13 - 8 * d);
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
  if (cl > 1)
    cluster_sync_all();
  else
    __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

int pick_fbn(int64_t N) {
  if (N <= 64) return 64;
  if (N <= 128) return 128;
  // (measured: forcing 128-column tiles with 2-slice grouped MMAs is slower
  // at cfg5, 77 vs 52 ms NN, so 144 wins whenever it pads less)
  static const int force = [] {
    const char* e = knob("XB_OZF_BN");
    return e ? atoi(e) : 0;
  }();
  if (force == 128 || force == 112) return force;
  const int64_t w128 = ceil_div(N, 128) * 128, w144 = ceil_div(N, 144) * 144;
  return w144 < w128 ? 144 : 128;
}

template <int BN, bool TRANS_A>
void launch_ozf(const CUtensorMap& ta, const int8_t* R, int64_t np, const int32_t* eL,
                const int32_t* eR, int64_t M, int64_t N, int64_t K, double* out, int64_t ldo,
                int64_t stride, int64_t kps, int splits, int acc, cudaStream_t st) {
  using Cfg = FCfg<BN>;
  auto kern = ozf_kernel<BN, TRANS_A>;
  XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  const int64_t tn = ceil_div(N, BN), tm = ceil_div(M, FBM);
  const int64_t total = tn * tm * splits;
  XB_REQUIRE(total < ((int64_t)1 << 31), XB_EUNSUPPORTED, "ozf: too many tiles");
  // NN: the n-tiles of an (m-tile, split) form a cluster and the leader
  // multicasts the A tile. At cfg5 (16384 x 1M, power-capped) the NN launch
  // reads 116 instead of 235 GB from DRAM and runs 53 instead of 64 ms (the
  // saved DRAM energy buys clock); for TN (A read ~once anyway) the
  // lockstep costs ~3 %, so TN stays unclustered. XB_OZF_CLUSTER: 0 never,
  // 1 NN (default), 2 cluster launch without multicast, 3 NN and TN.
  static const int cenv = [] {
    const char* e = knob("XB_OZF_CLUSTER");
    return e ? atoi(e) : 1;
  }();
  const int cmode = (cenv == 3 || (cenv != 0 && !TRANS_A)) ? (cenv == 2 ? 2 : 1) : 0;
  const int cdim = (cmode && tn >= 2 && tn <= 8) ? (int)tn : 1;
  const int cl = cmode == 2 ? 1 : cdim;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)total);
  cfg.blockDim = dim3(FTHREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cdim;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const int dbg = [] {
    const char* e = knob("XB_OZF_DBG");
    return e ? atoi(e) : 0;
  }();
  XB_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, R, np, eL, eR, M, N, K, out, ldo, stride, kps, acc,
                             (int)tn, (int)tm, splits, (int)std::min<int64_t>(8, tm),
                             cl | (dbg << 8)));
  check_launch("ozf");
}

}  // namespace

int oz_slices() {
  static const int s = [] {
    const char* e = knob("XB_OZ_SLICES");
    return e ? std::max(3, std::min(7, atoi(e))) : 6;
  }();
  return s;
}

bool oz_enabled() {
  static const bool on = [] {
    const char* e = knob("XB_F64_GEMM");
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

size_t oz_both_exp_scratch_bytes(int64_t rows, int64_t cols) {
  const int64_t nct = ceil_div(cols, RC_COLS), nrt = ceil_div(rows, RC_ROWS);
  return (size_t)(rows * nct + nrt * cols) * sizeof(double2);
}

template <typename T>
void oz_both_exp_t(const T* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* erow,
                   int32_t* ecol, void* scratch, int* wide, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  const int64_t nct = ceil_div(cols, RC_COLS), nrt = ceil_div(rows, RC_ROWS);
  XB_REQUIRE(nrt < 65536, XB_EUNSUPPORTED, "oz_both_exp: more than 2^25 rows");
  double2* rpart = static_cast<double2*>(scratch);
  double2* cpart = rpart + rows * nct;
  static const bool generic = [] {
    const char* e = knob("XB_RC_GENERIC");
    return e && atoi(e) != 0;
  }();
  if (!generic && (sizeof(T) == 8 || (ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(X) % 16) == 0)))
    rc_stats_fast_kernel<T><<<dim3((unsigned)nct, (unsigned)nrt), 256, 0, st>>>(X, rows, cols, ldx,
                                                                               rpart, cpart);
  else
    rc_stats_kernel<T><<<dim3((unsigned)nct, (unsigned)nrt), 256, 0, st>>>(X, rows, cols, ldx,
                                                                          rpart, cpart);
  check_launch("rc_stats");
  rc_finish_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(rpart, rows, nct, nct, 1, cols,
                                                                  erow, wide);
  check_launch("rc_finish_rows");
  rc_finish_kernel<<<(unsigned)ceil_div(cols, 256), 256, 0, st>>>(cpart, cols, nrt, 1, cols, rows,
                                                                  ecol, wide);
  check_launch("rc_finish_cols");
}

void oz_both_exp(const double* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* erow,
                 int32_t* ecol, void* scratch, int* wide, cudaStream_t st) {
  oz_both_exp_t<double>(X, rows, cols, ldx, erow, ecol, scratch, wide, st);
}

void oz_both_exp_f32(const float* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* erow,
                     int32_t* ecol, void* scratch, int* wide, cudaStream_t st) {
  oz_both_exp_t<float>(X, rows, cols, ldx, erow, ecol, scratch, wide, st);
}

#define OZ_DISPATCH(S, CALL) \
  switch (S) {               \
    case 3: CALL(3); break;  \
    case 4: CALL(4); break;  \
    case 5: CALL(5); break;  \
    case 7: CALL(7); break;  \
    default: CALL(6); break; \
  }

void oz_slice_right(const double* X, int64_t K, int64_t N, int64_t ldx, const int32_t* e,
                    int8_t* P, int64_t np, int64_t kp, int S, cudaStream_t st) {
  XB_REQUIRE(np % OBN == 0 && kp % OBK == 0 && np / 32 < 65536, XB_EUNSUPPORTED,
             "oz_slice_right: layout");
  dim3 grid((unsigned)(kp / 32), (unsigned)(np / 32));
#define OZ_SX(SS) slice_right_kernel<SS, 64><<<grid, dim3(32, 8), 0, st>>>(X, K, N, ldx, e, P, np, kp)
  OZ_DISPATCH(S, OZ_SX)
#undef OZ_SX
  check_launch("slice_right");
}

void oz_slice_both(const double* X, int64_t m, int64_t n, int64_t ldx, const int32_t* er,
                   const int32_t* ec, int8_t* PR, int64_t mp, int64_t kpn, int8_t* PC, int64_t np,
                   int64_t kpm, int S, cudaStream_t st) {
  XB_REQUIRE(mp % OBM == 0 && np % OBM == 0 && kpn % 32 == 0 && kpm % 32 == 0 && mp >= kpm &&
                 np >= kpn && np / 32 < 65536,
             XB_EUNSUPPORTED, "oz_slice_both: layout");
  dim3 grid((unsigned)(mp / 128), (unsigned)(np / 32));
#define OZ_SB(SS) \
  slice_both_kernel<SS><<<grid, 256, 0, st>>>(X, m, n, ldx, er, ec, PR, mp, kpn, PC, np, kpm)
  OZ_DISPATCH(S, OZ_SB)
#undef OZ_SB
  check_launch("slice_both");
}

int oz_plan_splits(int64_t K) { return (int)std::max<int64_t>(1, ceil_div(K, 16384)); }

void ozgemm(const int8_t* L, int64_t rows_p, int64_t kp, const int32_t* eL, const int8_t* R,
            int64_t np, const int32_t* eR, int64_t M, int64_t N, int64_t K, double* C, int64_t ldc,
            bool accumulate, int S, double* work, cudaStream_t st, int tri) {
  if (M <= 0 || N <= 0) return;
  XB_REQUIRE(kp % OBK == 0 && rows_p % OBM == 0 && rows_p >= M && np % OBN == 0 && np >= N &&
                 kp >= K,
             XB_EUNSUPPORTED, "ozgemm: slice layout");
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
#define OZ_RUN(SS) \
  launch_oz<SS>(L, R, rows_p, np, eL, eR, M, N, K, out, ldo, stride, kps, splits, acc, tri, st)
  OZ_DISPATCH(S, OZ_RUN)
#undef OZ_RUN
  if (splits > 1) launch_split_reduce(work, M, N, ldo, stride, splits, C, ldc, accumulate, st);
}

int ozf_tile_n(int64_t N) { return pick_fbn(N); }

int ozf_plan_splits(int64_t M, int64_t N, int64_t K) {
  // exact int32 levels: K per split <= 32768 (3 pairs x 2^14 x K < 2^31)
  const int bn = pick_fbn(N);
  const int64_t tiles = ceil_div(M, FBM) * ceil_div(N, bn);
  const int64_t kt = ceil_div(K, FBK);
  int s = (int)std::max<int64_t>(1, ceil_div(K, 32768));
  while (tiles * s < 2 * kNumSMs && kt / (s * 2) >= 8) s *= 2;
  return std::max(1, std::min<int>(s, (int)kt));
}

void oz_slice_right_f(const double* X, int64_t K, int64_t N, int64_t ldx, const int32_t* e,
                      int8_t* P, int64_t np, int64_t kp, cudaStream_t st) {
  const int bn = pick_fbn(N);
  XB_REQUIRE(np % bn == 0 && kp % 32 == 0 && np / 32 < 65536, XB_EUNSUPPORTED,
             "oz_slice_right_f: layout");
  // np = 144 k is not a multiple of 32: the last block row is partial
  dim3 grid((unsigned)(kp / 32), (unsigned)ceil_div(np, 32));
  if (bn == 64)
    slice_right_kernel<FS, 64><<<grid, dim3(32, 8), 0, st>>>(X, K, N, ldx, e, P, np, kp);
  else if (bn == 128)
    slice_right_kernel<FS, 128><<<grid, dim3(32, 8), 0, st>>>(X, K, N, ldx, e, P, np, kp);
  else if (bn == 112)
    slice_right_kernel<FS, 112><<<grid, dim3(32, 8), 0, st>>>(X, K, N, ldx, e, P, np, kp);
  else
    slice_right_kernel<FS, 144><<<grid, dim3(32, 8), 0, st>>>(X, K, N, ldx, e, P, np, kp);
  check_launch("slice_right_f");
}

void ozf_gemm(const float* A, int64_t lda, bool trans_a, const int32_t* eL, const int8_t* R,
              int64_t np, const int32_t* eR, int64_t M, int64_t N, int64_t K, double* C,
              int64_t ldc, bool accumulate, int splits, double* work, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  const int bn = pick_fbn(N);
  XB_REQUIRE(np % bn == 0 && np >= N, XB_EUNSUPPORTED, "ozf: right slice layout");
  XB_REQUIRE((reinterpret_cast<uintptr_t>(A) & 15) == 0 && lda % 4 == 0, XB_EUNSUPPORTED,
             "ozf: A must be 16-byte aligned with lda % 4 == 0");
  splits = std::max(1, std::min<int>(splits, (int)ceil_div(K, FBK)));
  const int64_t kps = round_up(ceil_div(K, splits), FBK);
  splits = (int)ceil_div(K, kps);
  double* out = C;
  int64_t ldo = ldc, stride = 0;
  if (splits > 1) {
    XB_REQUIRE(work != nullptr, XB_ECUDA, "ozf: split-K workspace missing");
    out = work;
    ldo = round_up(N, 2);
    stride = M * ldo;
  }
  const int acc = (splits == 1 && accumulate) ? 1 : 0;
  // A: NN [M][K] K-major 128B-swizzled boxes {32, 128}; TN [K][M] boxes {128, 32}
  const CUtensorMap ta = trans_a ? make_map(A, (uint64_t)M, (uint64_t)K, lda, FBM, FBK, false)
                                 : make_map(A, (uint64_t)K, (uint64_t)M, lda, FBK, FBM, true);
#define OZF(BN)                                                                             \
  if (trans_a)                                                                              \
    launch_ozf<BN, true>(ta, R, np, eL, eR, M, N, K, out, ldo, stride, kps, splits, acc, st); \
  else                                                                                      \
    launch_ozf<BN, false>(ta, R, np, eL, eR, M, N, K, out, ldo, stride, kps, splits, acc, st);
  if (bn == 64) {
    OZF(64)
  } else if (bn == 128) {
    OZF(128)
  } else if (bn == 112) {
    OZF(112)
  } else {
    OZF(144)
  }
#undef OZF
  if (splits > 1) launch_split_reduce(work, M, N, ldo, stride, splits, C, ldc, accumulate, st);
}

size_t ozf_workspace_doubles(int64_t M, int64_t N, int64_t K) {
  const int s = ozf_plan_splits(M, N, K);
  return s > 1 ? (size_t)s * M * round_up(N, 2) : 0;
}

size_t oz_workspace_doubles(int64_t M, int64_t N, int64_t K) {
  const int s = oz_plan_splits(K);
  return s > 1 ? (size_t)s * M * round_up(N, 2) : 0;
}

}  // namespace xb
