// FP64 tensor-core (DMMA) tile GEMM for the rSVD products.
//
// Replaces the reference's dense block_multiply (kernels.py:145-193,
// _cell_accumulate 80-84) for the product shapes of the hot path:
//   NN  Y  = A * X        A m x n row-major (K-contiguous), X n x l
//   TN  Z  = A^T * Q      A m x n row-major read as its transposed view
//                         (pool.py:390-418), reduce over the long m
//   TN  G  = Y^T * Y      the CholQR Gram (kernels.py:315-325 replacement)
// FP64 has no tcgen05 kind on sm_100a (ptxas rejects kind::f64),
// so the tensor-core path for f64 is the legacy mma.sync.m8n8k4.f64 (SASS
// DMMA). Operands stream global -> shared with cp.async (LDGSTS) in a
// STAGES-deep ring; every CTA owns a BM x BN output tile with BN covering
// the whole (padded) sketch width l, so each A element is read from HBM
// exactly once per product. Long reductions (TN over m, NN over n when the
// output tile count is below the SM count) are split over `splits` slices
// written to a workspace and summed in slice order by a second kernel — a
// fixed order, so results are deterministic run to run (no fp atomics).
//
// A may be float64 or float32 (Precision.SINGLE storage): a float32 A tile
// is widened to f64 in registers at fragment load, so products over f32
// inputs run with f64 accumulation (more accurate than the reference's f32
// compute dtype, core.py:43-46).
//
// Shared-memory layout: tile row strides are padded so the per-lane
// fragment loads of m8n8k4 (row = lane>>2, col = lane&3) are bank-conflict
// free: S = 4 (mod 8) elements for 8-byte tiles and K-contiguous 4-byte
// tiles, S = 8 (mod 16) for M-contiguous 4-byte tiles.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace xb {
namespace {

constexpr int pad_to(int x, int mod, int rem) { return x + ((rem - (x % mod)) % mod + mod) % mod; }

template <typename TA, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool TRANS_A>
struct DCfg {
  static constexpr int kThreads = WARPS_M * WARPS_N * 32;
  static constexpr int WM = BM / WARPS_M;  // rows per warp
  static constexpr int WN = BN / WARPS_N;  // cols per warp
  static constexpr int FM = WM / 8;        // 8x8 fragments per warp (M)
  static constexpr int FN = WN / 8;        // (N)
  static_assert(WM % 8 == 0 && WN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(BK % 4 == 0, "BK multiple of 4");
  static constexpr bool kF32 = sizeof(TA) == 4;
  // A tile: NN -> BM rows x BK (K-contig), TN -> BK rows x BM (M-contig)
  static constexpr int SA = TRANS_A ? (kF32 ? pad_to(BM, 16, 8) : pad_to(BM, 8, 4)) : pad_to(BK, 8, 4);
  static constexpr int A_ELEMS = TRANS_A ? BK * SA : BM * SA;
  static constexpr size_t A_BYTES = ((size_t)A_ELEMS * sizeof(TA) + 15) / 16 * 16;
  static constexpr int SB = pad_to(BN, 8, 4);
  static constexpr int B_ELEMS = BK * SB;
  static constexpr size_t STAGE_BYTES = A_BYTES + (size_t)B_ELEMS * sizeof(double);
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Async copies with zero fill of the bytes past src_bytes.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(dst)), "l"(src),
               "n"(BYTES), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Load a ROWS x COLS sub-block (global row-major, ld) into shared (stride S),
// zero-filling outside [row_lim, col_lim). VEC16 requires ld and col0 to be
// multiples of 16/sizeof(T) and a 16B-aligned base.
template <typename T, int ROWS, int COLS, int S, int NT, bool VEC16>
__device__ __forceinline__ void load_tile(T* sdst, const T* __restrict__ g, int64_t ld, int64_t row0,
                                          int64_t col0, int64_t row_lim, int64_t col_lim, int tid) {
  if constexpr (VEC16) {
    constexpr int E = 16 / sizeof(T);  // elements per 16B chunk
    constexpr int CPR = COLS / E;
    static_assert(COLS % E == 0, "tile width must hold whole 16B chunks");
    constexpr int TOTAL = ROWS * CPR;
#pragma unroll
    for (int i = tid; i < TOTAL; i += NT) {
      const int r = i / CPR;
      const int c = (i - r * CPR) * E;
      const int64_t gr = row0 + r, gc = col0 + c;
      const T* src = g;
      int bytes = 0;
      if (gr < row_lim && gc < col_lim) {
        src = g + gr * ld + gc;
        const int64_t left = col_lim - gc;
        bytes = (int)(left >= E ? 16 : left * (int64_t)sizeof(T));
      }
      cp_async16(sdst + r * S + c, src, bytes);
    }
  } else {
    constexpr int TOTAL = ROWS * COLS;
#pragma unroll 4
    for (int i = tid; i < TOTAL; i += NT) {
      const int r = i / COLS;
      const int c = i - r * COLS;
      const int64_t gr = row0 + r, gc = col0 + c;
      const T* src = g;
      int bytes = 0;
      if (gr < row_lim && gc < col_lim) {
        src = g + gr * ld + gc;
        bytes = sizeof(T);
      }
      cp_async_small<sizeof(T)>(sdst + r * S + c, src, bytes);
    }
  }
}

// C (or the split slice of the workspace) = op(A) * B over k in
// [z * k_per_split, min(K, (z+1) * k_per_split)).
template <typename TA, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool TRANS_A,
          bool A16, bool B16>
__global__ void __launch_bounds__(WARPS_M* WARPS_N * 32, 1)
    dgemm_kernel(int64_t M, int64_t N, int64_t K, const TA* __restrict__ A, int64_t lda,
                 const double* __restrict__ B, int64_t ldb, double* __restrict__ C, int64_t ldc,
                 int64_t split_stride, int64_t k_per_split, int accumulate, int tri) {
  using Cfg = DCfg<TA, BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * BN;
  // tri 1: tiles strictly below the diagonal are never read (SYRK-like Gram)
  if (tri == 1 && m0 > n0 + BN - 1) return;
  const int64_t kbeg = (int64_t)blockIdx.z * k_per_split;
  int64_t kend = min(K, kbeg + k_per_split);
  // tri 2: B upper triangular, rows k >= n0 + BN of this N-tile are zero
  if (tri == 2) kend = min(kend, n0 + BN);
  C += (int64_t)blockIdx.z * split_stride;

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int ktiles = kend > kbeg ? (int)ceil_div(kend - kbeg, BK) : 0;

  auto stage_a = [&](int stage) {
    return reinterpret_cast<TA*>(smem_raw + (size_t)stage * Cfg::STAGE_BYTES);
  };
  auto stage_b = [&](int stage) {
    return reinterpret_cast<double*>(smem_raw + (size_t)stage * Cfg::STAGE_BYTES + Cfg::A_BYTES);
  };
  auto load_stage = [&](int stage, int kt) {
    const int64_t k0 = kbeg + (int64_t)kt * BK;
    if constexpr (TRANS_A) {
      load_tile<TA, BK, BM, Cfg::SA, Cfg::kThreads, A16>(stage_a(stage), A, lda, k0, m0, kend, M, tid);
    } else {
      load_tile<TA, BM, BK, Cfg::SA, Cfg::kThreads, A16>(stage_a(stage), A, lda, m0, k0, M, kend, tid);
    }
    load_tile<double, BK, BN, Cfg::SB, Cfg::kThreads, B16>(stage_b(stage), B, ldb, k0, n0, kend, N, tid);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const TA* sA = stage_a(kt % STAGES);
    const double* sB = stage_b(kt % STAGES);
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[Cfg::FM], bf[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) {
        const int row = wm * Cfg::WM + i * 8 + g;  // output row within tile
        if constexpr (TRANS_A)
          af[i] = (double)sA[(ks * 4 + t) * Cfg::SA + row];
        else
          af[i] = (double)sA[row * Cfg::SA + ks * 4 + t];
      }
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        const int col = wn * Cfg::WN + j * 8 + g;
        bf[j] = sB[(ks * 4 + t) * Cfg::SB + col];
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue: fragment (row g, cols 2t, 2t+1) of each 8x8 block.
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) {
    const int64_t r = m0 + wm * Cfg::WM + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
      const int64_t c = n0 + wn * Cfg::WN + j * 8 + 2 * t;
      double* dst = C + r * ldc + c;
      if (c + 1 < N && ((ldc & 1) == 0)) {
        double2 v = make_double2(acc[i][j][0], acc[i][j][1]);
        if (accumulate) {
          const double2 o = *reinterpret_cast<const double2*>(dst);
          v.x += o.x;
          v.y += o.y;
        }
        *reinterpret_cast<double2*>(dst) = v;
      } else {
        if (c < N) dst[0] = accumulate ? dst[0] + acc[i][j][0] : acc[i][j][0];
        if (c + 1 < N) dst[1] = accumulate ? dst[1] + acc[i][j][1] : acc[i][j][1];
      }
    }
  }
}

// out[r, c] = sum_{s < S} work[s][r, c] in slice order.
__global__ void split_reduce_kernel(const double* __restrict__ work, int64_t M, int64_t N,
                                    int64_t ldw, int64_t stride, int S, double* __restrict__ C,
                                    int64_t ldc, int accumulate) {
  const int64_t total = M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / N, c = idx - r * N;
    const double* p = work + r * ldw + c;
    double acc = p[0];
    for (int s = 1; s < S; ++s) acc += p[s * stride];
    C[r * ldc + c] = accumulate ? C[r * ldc + c] + acc : acc;
  }
}

// Many slices, few outputs (the CholQR Gram: l x l outputs, ~300 slices):
// a block owns 32 consecutive outputs, its 8 warps stride the slices, and
// warp partials are combined in warp order — a fixed order, deterministic.
__global__ void __launch_bounds__(256) split_reduce_wide_kernel(
    const double* __restrict__ work, int64_t M, int64_t N, int64_t ldw, int64_t stride, int S,
    double* __restrict__ C, int64_t ldc, int accumulate) {
  __shared__ double part[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t idx = (int64_t)blockIdx.x * 32 + lane;
  const int64_t total = M * N;
  double acc = 0.0;
  int64_t r = 0, c = 0;
  if (idx < total) {
    r = idx / N;
    c = idx - r * N;
    const double* p = work + r * ldw + c;
    for (int s = warp; s < S; s += 8) acc += p[(int64_t)s * stride];
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && idx < total) {
    double sum = part[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) sum += part[w][lane];
    C[r * ldc + c] = accumulate ? C[r * ldc + c] + sum : sum;
  }
}

}  // namespace

// ---- dispatch ----------------------------------------------------------------

namespace {

template <typename TA, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, bool TRANS_A>
void run_cfg(const DGemmArgs& g, int splits, int64_t k_per_split, double* out, int64_t ldo,
             int64_t split_stride, cudaStream_t st) {
  using Cfg = DCfg<TA, BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A>;
  constexpr int64_t E = 16 / sizeof(TA);
  const TA* A = static_cast<const TA*>(g.A);
  const bool a16 = (g.lda % E == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  const bool b16 = ((g.ldb & 1) == 0) && ((reinterpret_cast<uintptr_t>(g.B) & 15) == 0);
  dim3 grid((unsigned)ceil_div(g.M, BM), (unsigned)ceil_div(g.N, BN), (unsigned)splits);
  auto launch = [&](auto kernel) {
    XB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Cfg::SMEM));
    // with split-K the slices go to the workspace and the reduce accumulates
    const int acc_here = (splits == 1 && g.accumulate) ? 1 : 0;
    kernel<<<grid, Cfg::kThreads, Cfg::SMEM, st>>>(g.M, g.N, g.K, A, g.lda, g.B, g.ldb, out, ldo,
                                                   split_stride, k_per_split, acc_here, g.tri);
    check_launch("dgemm");
  };
  if (a16 && b16)
    launch(dgemm_kernel<TA, BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A, true, true>);
  else if (a16)
    launch(dgemm_kernel<TA, BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A, true, false>);
  else if (b16)
    launch(dgemm_kernel<TA, BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A, false, true>);
  else
    launch(dgemm_kernel<TA, BM, BN, BK, WARPS_M, WARPS_N, STAGES, TRANS_A, false, false>);
}

// Tile width for the N (sketch) dimension: the whole padded l in one tile
// when it fits, so A streams once.
int pick_bn(int64_t N) {
  if (N <= 32) return 32;
  if (N <= 64) return 64;
  if (N == 120) return 120;
  if (N <= 112) return 112;
  if (N <= 128) return 128;
  // wide sketches (cfg4 l=220 -> 224 = 2 x 112, cfg5 l=550 -> 552 in 5 x 112):
  // the tile width that wastes the fewest padded columns
  const int64_t w112 = ceil_div(N, 112) * 112, w128 = ceil_div(N, 128) * 128;
  return w112 < w128 ? 112 : 128;
}

// Tile variants. The l = 120 products over A (cfg2's hot shape) have
// alternatives selectable with XB_DGEMM_VARIANT for tuning runs (measured
// on B200, tools/tune_gemm.py: BK=32/3 stages is the fastest); everything
// else uses the BK=16 / 4-stage tile.
struct Variant {
  int id, BM, BK, ctas_per_sm;
};

Variant pick_variant(const DGemmArgs& g) {
  const int bn = pick_bn(g.N);
  int v = 0;
  if (bn == 120 && g.K >= 4096 && !g.a_f32) {
    static const int env = [] {
      const char* e = knob("XB_DGEMM_VARIANT");
      return e ? atoi(e) : -1;
    }();
    v = env >= 0 ? env : 1;
  }
  switch (v) {
    case 1: return {1, 128, 32, 1};
    case 2: return {2, 64, 16, 2};
    case 3: return {3, 128, 16, 1};
    default: return {0, 128, 16, 1};
  }
}

int64_t kper(int64_t K, int splits, int bk) { return round_up(ceil_div(K, splits), bk); }

template <typename TA, bool TRANS_A>
void dispatch(const DGemmArgs& g, const Variant& var, int splits, int64_t kps, double* out,
              int64_t ldo, int64_t stride, cudaStream_t st) {
  const int bn = pick_bn(g.N);
  if constexpr (std::is_same<TA, double>::value) {
    if (bn == 120) {
      switch (var.id) {
        case 1: run_cfg<TA, 128, 120, 32, 4, 3, 3, TRANS_A>(g, splits, kps, out, ldo, stride, st); return;
        case 2: run_cfg<TA, 64, 120, 16, 2, 3, 4, TRANS_A>(g, splits, kps, out, ldo, stride, st); return;
        case 3: run_cfg<TA, 128, 120, 16, 2, 3, 4, TRANS_A>(g, splits, kps, out, ldo, stride, st); return;
        default: run_cfg<TA, 128, 120, 16, 4, 3, 4, TRANS_A>(g, splits, kps, out, ldo, stride, st); return;
      }
    }
  }
  switch (bn) {
    case 32: run_cfg<TA, 128, 32, 16, 4, 1, 4, TRANS_A>(g, splits, kps, out, ldo, stride, st); break;
    case 64: run_cfg<TA, 128, 64, 16, 4, 2, 4, TRANS_A>(g, splits, kps, out, ldo, stride, st); break;
    case 112: run_cfg<TA, 128, 112, 16, 4, 2, 4, TRANS_A>(g, splits, kps, out, ldo, stride, st); break;
    default: run_cfg<TA, 128, 128, 16, 4, 4, 4, TRANS_A>(g, splits, kps, out, ldo, stride, st); break;
  }
}

}  // namespace

void launch_split_reduce(const double* work, int64_t M, int64_t N, int64_t ldw, int64_t stride,
                         int S, double* C, int64_t ldc, bool accumulate, cudaStream_t st) {
  const int64_t total = M * N;
  if (S >= 16) {
    split_reduce_wide_kernel<<<(unsigned)ceil_div(total, 32), 256, 0, st>>>(
        work, M, N, ldw, stride, S, C, ldc, accumulate ? 1 : 0);
  } else {
    int blocks = (int)std::min<int64_t>(ceil_div(total, 256), kNumSMs * 8);
    split_reduce_kernel<<<blocks, 256, 0, st>>>(work, M, N, ldw, stride, S, C, ldc,
                                                accumulate ? 1 : 0);
  }
  check_launch("split_reduce");
}

int dgemm_plan_splits(const DGemmArgs& g) {
  const Variant var = pick_variant(g);
  const int64_t tiles = ceil_div(g.M, var.BM) * ceil_div(g.N, pick_bn(g.N));
  const int64_t kt = ceil_div(g.K, var.BK);
  const int64_t slots = (int64_t)kNumSMs * var.ctas_per_sm;
  // Fill the machine: aim for >= ~6 waves, but keep at least 8 k-tiles per
  // slice so the pipeline has something to hide.
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 256; ++s) {
    if (kt / s < 8 && s > 1) break;
    const int64_t ctas = tiles * s;
    const int64_t waves = ceil_div(ctas, slots);
    const double eff = (double)ctas / (double)(waves * slots);
    // prefer fewer slices unless the wave efficiency improves materially
    if (eff > best_eff + 0.03) {
      best_eff = eff;
      best = s;
    }
    if (ctas >= 6 * slots && eff > 0.95) break;
  }
  // Tiny outputs (Gram: one tile) need many slices to use the machine.
  if (tiles <= 4) best = (int)std::min<int64_t>(std::max<int64_t>(1, kt / 8), 2 * kNumSMs / tiles);
  return std::max(1, best);
}

size_t dgemm_workspace_doubles(const DGemmArgs& g, int splits) {
  if (splits <= 1) return 0;
  return (size_t)splits * (size_t)g.M * (size_t)round_up(g.N, 2);
}

void dgemm(const DGemmArgs& g, int splits, double* work, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  if (g.K <= 0) {
    if (!g.accumulate)
      for (int64_t r = 0; r < g.M; ++r)
        XB_CUDA(cudaMemsetAsync(g.C + r * g.ldc, 0, g.N * sizeof(double), st));
    return;
  }
  const Variant var = pick_variant(g);
  splits = std::max(1, std::min<int>(splits, (int)ceil_div(g.K, var.BK)));
  const int64_t kps = kper(g.K, splits, var.BK);
  splits = (int)ceil_div(g.K, kps);
  double* out = g.C;
  int64_t ldo = g.ldc, stride = 0;
  if (splits > 1) {
    XB_REQUIRE(work != nullptr, XB_ECUDA, "dgemm: split-K workspace missing");
    out = work;
    ldo = round_up(g.N, 2);
    stride = g.M * ldo;
  }
  if (g.a_f32) {
    if (g.trans_a)
      dispatch<float, true>(g, var, splits, kps, out, ldo, stride, st);
    else
      dispatch<float, false>(g, var, splits, kps, out, ldo, stride, st);
  } else {
    if (g.trans_a)
      dispatch<double, true>(g, var, splits, kps, out, ldo, stride, st);
    else
      dispatch<double, false>(g, var, splits, kps, out, ldo, stride, st);
  }
  if (splits > 1) {
    const int64_t total = g.M * g.N;
    if (splits >= 16) {
      split_reduce_wide_kernel<<<(unsigned)ceil_div(total, 32), 256, 0, st>>>(
          work, g.M, g.N, ldo, stride, splits, g.C, g.ldc, g.accumulate ? 1 : 0);
    } else {
      int blocks = (int)std::min<int64_t>(ceil_div(total, 256), kNumSMs * 8);
      split_reduce_kernel<<<blocks, 256, 0, st>>>(work, g.M, g.N, ldo, stride, splits, g.C, g.ldc,
                                                  g.accumulate ? 1 : 0);
    }
    check_launch("split_reduce");
  }
}

}  // namespace xb
