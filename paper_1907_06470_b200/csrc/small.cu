// l x l kernels of the hot path (single CTA, latency-bound, l <= ~160 in
// shared memory; larger l on cooperative multi-CTA grids over L2-resident
// global scratch).
//
//  chol_inv  G = R^T R (upper R, f64) and R^{-1}: the small step of CholQR2,
//            which replaces the reference's Householder thin_qr
//            (kernels.py:297-351). Right-looking, unscaled Schur updates with
//            ONE barrier per column; triangular inverse column by column
//            (LAPACK dtrti2 order) with warp-level dot products.
//  jacobi    one-sided Hestenes Jacobi SVD of M = R_B^T, replacing the
//            Golub-Kahan svd_small (kernels.py:542-562) on the projected
//            factor. Round-robin (circle) ordering: every round rotates l/2
//            disjoint column pairs in parallel, one 16-lane group per pair;
//            M's columns and the accumulated right rotations J both live in
//            shared memory when they fit. Output sorted descending (stable,
//            kernels.py:535) with the sign rule of kernels.py:556-561.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <vector>

#include "common.cuh"

namespace xb {
namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double warp_sum32(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    chol_inv_kernel(const double* __restrict__ G, int64_t ldg, int l, double tau,
                    double* __restrict__ R, double* __restrict__ Rinv, int64_t ldr,
                    int* __restrict__ flag, double* gw, int use_smem) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double diag0[1024];
  __shared__ double pivs[1024];
  double* W = use_smem ? sm : gw;
  // odd row stride (conflict-free column reads)
  const int64_t lw = l | 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // load the upper triangle (row-major, stride l); the strictly lower part
  // holds E = L^-1 (unit diagonal implied), zero at the start
  for (int i = warp; i < l; i += kWarps)
    for (int c = lane; c < l; c += 32) W[(int64_t)i * lw + c] = (c >= i) ? G[(int64_t)i * ldg + c] : 0.0;
  for (int j = tid; j < l; j += kThreads) diag0[j] = G[(int64_t)j * ldg + j];
  __syncthreads();
  // Symmetric elimination G = L D L^T, one barrier per column. Row i > j of
  // the trailing block loses f = W[j][i] / d_j times row j in its upper part
  // (columns >= i) and, in the same step, E = L^-1 gets the same row
  // operation in its lower part (columns <= j < i) — the two never overlap,
  // so the triangular inverse costs no extra pass or barrier:
  // R = D^-1/2 W, R^-1 = E^T D^-1/2.
  bool failed = false;
  for (int j = 0; j < l; ++j) {
    const double piv = W[(int64_t)j * lw + j];
    const bool ok = (piv > tau * diag0[j]) && (piv > 0.0);
    const double pe = ok ? piv : fmax(fabs(diag0[j]), DBL_MIN);  // keep going; result discarded
    failed |= !ok;
    if (tid == 0) pivs[j] = pe;
    const double inv = 1.0 / pe;
    const double* rowj = W + (int64_t)j * lw;
    for (int i = j + 1 + warp; i < l; i += kWarps) {
      const double f = rowj[i] * inv;
      double* rowi = W + (int64_t)i * lw;
      for (int c = i + lane; c < l; c += 32) rowi[c] -= f * rowj[c];
      for (int c = lane; c < j; c += 32) rowi[c] -= f * rowj[c];
      if (lane == 0) rowi[j] = -f;
    }
    __syncthreads();
  }
  if (failed && tid == 0) *flag = 1;
  // R[j][c] = W[j][c] / sqrt(d_j) (c >= j); R^-1[a][b] = E[b][a] / sqrt(d_b)
  for (int i = warp; i < l; i += kWarps) {
    const double rs = 1.0 / sqrt(pivs[i]);
    for (int c = lane; c < l; c += 32) {
      R[(int64_t)i * ldr + c] = (c >= i) ? W[(int64_t)i * lw + c] * rs : 0.0;
      double e = 0.0;
      if (c > i) e = W[(int64_t)c * lw + i] / sqrt(pivs[c]);
      else if (c == i) e = rs;
      Rinv[(int64_t)i * ldr + c] = e;
    }
  }
}

// ---------------------------------------------------------------------------
// The same factorisation in blocks of 8 pivots (shared-memory case, l <= ~160).
// chol_inv_kernel pays one CTA barrier and one FP64 reciprocal (~250 cycles)
// plus a chain of dependent row updates per pivot: ~2600 cycles per column at
// l = 120, 0.16 ms per call and eight calls per cfg2 step. In the symmetric
// row elimination the multiplier f_ij = W[j][i] / d_j of a trailing row i
// depends on the pivot row j alone, so the updates of row i by different
// pivots are independent and additive:
//   phase 1  the 8 rows of the block are eliminated among themselves by 8
//            warps (one per row; a named barrier per pivot), which makes the
//            block's pivot rows, pivots and reciprocals final;
//   phase 2  every trailing row takes all 8 pivots in one pass (rank-8
//            update of its upper part and of its E = L^-1 part), all warps.
// 15 block steps of one CTA barrier instead of 120 column steps, and phase 1
// of the next block overlapped with phase 2 of this one: 164 -> 135 us at
// l = 120 without the overlap. (A variant with the diagonal block on one warp, one thread per
// column for the block rows and a (row group, column) thread grid for the
// trailing update ran 166 us: profiles/r02_chol_inv_experiments.md.)
constexpr int kCB8 = 8;

__global__ void __launch_bounds__(kThreads, 1)
    chol_inv_blocked_kernel(const double* __restrict__ G, int64_t ldg, int l, double tau,
                            double* __restrict__ R, double* __restrict__ Rinv, int64_t ldr,
                            int* __restrict__ flag) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double diag0[256];
  __shared__ double pivs[256];
  __shared__ double invs[2][kCB8];
  __shared__ int s_failed;
  double* W = sm;
  const int64_t lw = l | 1;  // odd row stride (conflict-free column reads)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = warp; i < l; i += kWarps)
    for (int c = lane; c < l; c += 32) W[(int64_t)i * lw + c] = (c >= i) ? G[(int64_t)i * ldg + c] : 0.0;
  for (int j = tid; j < l; j += kThreads) diag0[j] = G[(int64_t)j * ldg + j];
  if (tid == 0) s_failed = 0;
  __syncthreads();
  // phase 1 of the block at j0 (warps 0 .. nb-1, one per row; reciprocals into
  // invs[buf])
  auto phase1 = [&](int j0, int nb, int buf) {
    const int i = j0 + warp;
    double* rowi = W + (int64_t)i * lw;
    for (int jj = 0; jj < nb; ++jj) {
      const int j = j0 + jj;
      const double* rowj = W + (int64_t)j * lw;
      const double piv = rowj[j];
      const bool ok = (piv > tau * diag0[j]) && (piv > 0.0);
      const double pe = ok ? piv : fmax(fabs(diag0[j]), DBL_MIN);  // keep going; result discarded
      const double inv = 1.0 / pe;
      if (warp == jj && lane == 0) {
        pivs[j] = pe;
        invs[buf][jj] = inv;
        if (!ok) s_failed = 1;
      }
      if (warp > jj) {
        const double f = rowj[i] * inv;
        for (int c = i + lane; c < l; c += 32) rowi[c] -= f * rowj[c];
        for (int c = lane; c < j; c += 32) rowi[c] -= f * rowj[c];
        if (lane == 0) rowi[j] = -f;
      }
      // the warps of the block only (row j + 1 is final for the next pivot)
      asm volatile("bar.sync 1, %0;\n" ::"r"(32 * nb) : "memory");
    }
  };
  // phase 2 of trailing row i for the block at j0
  auto phase2_row = [&](int i, int j0, int nb, int buf) {
    double* rowi = W + (int64_t)i * lw;
    double f[kCB8];
#pragma unroll
    for (int jj = 0; jj < kCB8; ++jj)
      f[jj] = jj < nb ? W[(int64_t)(j0 + jj) * lw + i] * invs[buf][jj] : 0.0;
    // upper part (c >= i) and the E part of earlier blocks (c < j0)
    for (int c = lane; c < l; c += 32) {
      if (c >= i || c < j0) {
        double a0 = rowi[c], a1 = 0.0;
#pragma unroll
        for (int jj = 0; jj < kCB8; jj += 2) {
          if (jj < nb) a0 = fma(-f[jj], W[(int64_t)(j0 + jj) * lw + c], a0);
          if (jj + 1 < nb) a1 = fma(-f[jj + 1], W[(int64_t)(j0 + jj + 1) * lw + c], a1);
        }
        rowi[c] = a0 + a1;
      }
    }
    // E entries inside the block: E_i[c] = -f_c - sum_{j > c in block} f_j E[j][c]
    if (lane < nb) {
      const int c = j0 + lane;
      double e = 0.0;
#pragma unroll
      for (int jj = 0; jj < kCB8; ++jj) {
        if (jj == lane) e -= f[jj];
        else if (jj > lane && jj < nb) e = fma(-f[jj], W[(int64_t)(j0 + jj) * lw + c], e);
      }
      rowi[c] = e;
    }
  };
  // Look-ahead: in block step J the first 8 warps update the NEXT block's rows
  // first and go straight on to that block's phase 1 while warps 8-31 update
  // the remaining trailing rows — phase 1 (a chain of 8 reciprocals) hides
  // behind phase 2.
  if (warp < min(kCB8, l)) phase1(0, min(kCB8, l), 0);
  __syncthreads();
  int buf = 0;
  for (int j0 = 0; j0 < l; j0 += kCB8, buf ^= 1) {
    const int nb = min(kCB8, l - j0);
    const int n1 = j0 + nb;              // first trailing row = the next block's first row
    const int nb1 = min(kCB8, l - n1);   // rows of the next block (<= 0: none)
    if (warp < kCB8) {
      if (warp < nb1) {
        phase2_row(n1 + warp, j0, nb, buf);
        asm volatile("bar.sync 1, %0;\n" ::"r"(32 * nb1) : "memory");
        phase1(n1, nb1, buf ^ 1);
      }
    } else {
      for (int i = n1 + kCB8 + (warp - kCB8); i < l; i += kWarps - kCB8)
        phase2_row(i, j0, nb, buf);
    }
    __syncthreads();
  }
  if (s_failed && tid == 0) *flag = 1;
  // R[j][c] = W[j][c] / sqrt(d_j) (c >= j); R^-1[a][b] = E[b][a] / sqrt(d_b)
  for (int i = warp; i < l; i += kWarps) {
    const double rs = 1.0 / sqrt(pivs[i]);
    for (int c = lane; c < l; c += 32) {
      R[(int64_t)i * ldr + c] = (c >= i) ? W[(int64_t)i * lw + c] * rs : 0.0;
      double e = 0.0;
      if (c > i) e = W[(int64_t)c * lw + i] / sqrt(pivs[c]);
      else if (c == i) e = rs;
      Rinv[(int64_t)i * ldr + c] = e;
    }
  }
}

// ---------------------------------------------------------------------------
// chol_coop: the same factorisation for sketch widths whose l x l matrix does
// not fit one CTA's shared memory (l > ~160; config 5: l = 550). A single CTA
// streaming the matrix through L2 one column at a time took ~18 ms at l = 550;
// this is a blocked (32-wide) right-looking Cholesky over a cooperative grid:
//   A  CTA 0 factors the diagonal block W_JJ = R_JJ^T R_JJ (pivot test as
//      above) and inverts it, D_J = R_JJ^{-1}
//   B  all CTAs: panel R_J,>J = D_J^T W_J,>J (one thread per column)
//   C  all CTAs: trailing update W_>J,>J -= R_J,>J^T R_J,>J (32 x 32 tiles)
// then R^{-1} by block diagonals: X_JJ = D_J, X_IJ = -D_I sum_{I<K<=J} R_IK X_KJ
// (all (I, I+d) blocks of one diagonal d in parallel). Indices >= l are padded
// with the identity. Scratch: W, X (lp x lp) and D (nb x 32 x 32), lp = 32 nb.
constexpr int kCB = 32;
constexpr int kCT = 256;

__global__ void __launch_bounds__(kCT)
    chol_coop_kernel(const double* __restrict__ G, int64_t ldg, int l, double tau,
                     double* __restrict__ R, double* __restrict__ Rinv, int64_t ldr,
                     int* __restrict__ flag, double* __restrict__ ws) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int nb = (l + kCB - 1) / kCB, lp = nb * kCB;
  double* W = ws;
  double* X = W + (int64_t)lp * lp;
  double* D = X + (int64_t)lp * lp;
  __shared__ double sa[kCB][kCB + 1], sb[kCB][kCB + 1], sc[kCB][kCB + 1];
  const int tid = threadIdx.x;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + tid;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t ll = (int64_t)lp * lp;
  const int tr = tid >> 3, tc = (tid & 7) * 4;  // tile coordinates: row, 4 columns

  for (int64_t idx = gt; idx < ll; idx += gthreads) {
    const int i = (int)(idx / lp), c = (int)(idx - (int64_t)i * lp);
    W[idx] = (i < l && c < l) ? (c >= i ? G[(int64_t)i * ldg + c] : 0.0) : (i == c ? 1.0 : 0.0);
  }
  grid.sync();

  for (int jb = 0; jb < nb; ++jb) {
    const int j0 = jb * kCB;
    // A: diagonal block (warp 0 of CTA 0; lane = column)
    if (blockIdx.x == 0 && tid < 32) {
      const int lane = tid;
      for (int r = 0; r < kCB; ++r) sa[r][lane] = W[(int64_t)(j0 + r) * lp + j0 + lane];
      __syncwarp();
      bool fail = false;
      for (int j = 0; j < kCB; ++j) {
        const double piv = sa[j][j];
        const int gi = j0 + j;
        const double d0 = gi < l ? G[(int64_t)gi * ldg + gi] : 1.0;
        const bool ok = (piv > tau * d0) && (piv > 0.0);
        const double pe = ok ? piv : fmax(fabs(d0), DBL_MIN);  // keep going; result discarded
        fail |= !ok;
        const double rjj = sqrt(pe);
        const double v = lane > j ? sa[j][lane] / rjj : (lane == j ? rjj : 0.0);
        __syncwarp();
        sa[j][lane] = v;
        __syncwarp();
        for (int i = j + 1; i < kCB; ++i)
          if (lane >= i) sa[i][lane] -= sa[j][i] * sa[j][lane];
        __syncwarp();
      }
      if (fail && lane == 0) *flag = 1;
      // column `lane` of R_JJ^{-1} (lane-private: no synchronisation inside)
      sb[lane][lane] = 1.0 / sa[lane][lane];
      for (int i = lane - 1; i >= 0; --i) {
        double acc = 0.0;
        for (int p = i + 1; p <= lane; ++p) acc += sa[i][p] * sb[p][lane];
        sb[i][lane] = -acc / sa[i][i];
      }
      for (int i = lane + 1; i < kCB; ++i) sb[i][lane] = 0.0;
      __syncwarp();
      for (int r = 0; r < kCB; ++r) {
        W[(int64_t)(j0 + r) * lp + j0 + lane] = lane >= r ? sa[r][lane] : 0.0;
        D[(int64_t)jb * kCB * kCB + r * kCB + lane] = sb[r][lane];
      }
    }
    grid.sync();
    // B: panel rows j0.., columns beyond the block: x = D_J^T w
    const int ncols = lp - j0 - kCB;
    const double* Dj = D + (int64_t)jb * kCB * kCB;
    for (int64_t cc = gt; cc < ncols; cc += gthreads) {
      const int c = j0 + kCB + (int)cc;
      double w[kCB];
#pragma unroll
      for (int s2 = 0; s2 < kCB; ++s2) w[s2] = W[(int64_t)(j0 + s2) * lp + c];
#pragma unroll
      for (int r = 0; r < kCB; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int s2 = 0; s2 <= r; ++s2) acc += __ldg(&Dj[s2 * kCB + r]) * w[s2];
        W[(int64_t)(j0 + r) * lp + c] = acc;
      }
    }
    grid.sync();
    // C: trailing tiles (a <= b) of the blocks after jb
    const int n = nb - jb - 1;
    const int tiles = n * (n + 1) / 2;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int a = 0, rem = t;
      while (rem >= n - a) {
        rem -= n - a;
        ++a;
      }
      const int b = a + rem;
      const int ci = (jb + 1 + a) * kCB, cb = (jb + 1 + b) * kCB;
      for (int e = tid; e < kCB * kCB; e += kCT) {
        const int r = e >> 5, x = e & 31;
        sa[r][x] = W[(int64_t)(j0 + r) * lp + ci + x];
        sb[r][x] = W[(int64_t)(j0 + r) * lp + cb + x];
      }
      __syncthreads();
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
      for (int s2 = 0; s2 < kCB; ++s2) {
        const double ar = sa[s2][tr];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += ar * sb[s2][tc + q];
      }
      double* dst = W + (int64_t)(ci + tr) * lp + cb + tc;
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] -= acc[q];
      __syncthreads();
    }
    grid.sync();
  }

  // R^{-1} by block diagonals
  for (int64_t idx = gt; idx < ll; idx += gthreads) {
    const int i = (int)(idx / lp), c = (int)(idx - (int64_t)i * lp);
    const int bi = i / kCB, bc = c / kCB;
    X[idx] = bi == bc ? D[(int64_t)bi * kCB * kCB + (i % kCB) * kCB + (c % kCB)] : 0.0;
  }
  grid.sync();
  for (int d = 1; d < nb; ++d) {
    for (int t = blockIdx.x; t < nb - d; t += gridDim.x) {
      const int I = t, J = t + d;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int K = I + 1; K <= J; ++K) {
        for (int e = tid; e < kCB * kCB; e += kCT) {
          const int r = e >> 5, x = e & 31;
          sa[r][x] = W[(int64_t)(I * kCB + r) * lp + K * kCB + x];
          sb[r][x] = X[(int64_t)(K * kCB + r) * lp + J * kCB + x];
        }
        __syncthreads();
#pragma unroll 8
        for (int p = 0; p < kCB; ++p) {
          const double ar = sa[tr][p];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] += ar * sb[p][tc + q];
        }
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) sc[tr][tc + q] = acc[q];
      for (int e = tid; e < kCB * kCB; e += kCT) sa[e >> 5][e & 31] = D[(int64_t)I * kCB * kCB + e];
      __syncthreads();
      double out[4] = {0.0, 0.0, 0.0, 0.0};
      for (int p = tr; p < kCB; ++p) {
        const double ar = sa[tr][p];
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q] -= ar * sc[p][tc + q];
      }
      double* dst = X + (int64_t)(I * kCB + tr) * lp + J * kCB + tc;
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = out[q];
      __syncthreads();
    }
    grid.sync();
  }
  for (int64_t idx = gt; idx < (int64_t)l * l; idx += gthreads) {
    const int i = (int)(idx / l), c = (int)(idx - (int64_t)i * l);
    R[(int64_t)i * ldr + c] = c >= i ? W[(int64_t)i * lp + c] : 0.0;
    Rinv[(int64_t)i * ldr + c] = c >= i ? X[(int64_t)i * lp + c] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Jacobi. X (l x l, column-major: X[c*l + r]) = M = R^T, i.e. X[:, c] = R[c, :].
// J (column-major) in shared memory (j_in_smem) or global `gj`.
constexpr int kGroup = 16;                    // lanes per column pair
constexpr int kGroups = kThreads / kGroup;    // 64 pairs in flight per round

// Sum over the 16 lanes of this half-warp. The mask names only this half:
// the other half may be idle (odd l, dummy pair) or on a different pair.
__device__ __forceinline__ void group_sum3(double& a, double& b, double& c) {
  const unsigned mask = (threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu;
#pragma unroll
  for (int o = kGroup / 2; o > 0; o >>= 1) {
    a += __shfl_xor_sync(mask, a, o);
    b += __shfl_xor_sync(mask, b, o);
    c += __shfl_xor_sync(mask, c, o);
  }
}

// Single-CTA Jacobi tail: singular values = column norms of X, stable
// descending order, U_B columns sign-fixed (largest |entry| positive,
// earliest row on ties, kernels.py:556-561), W_k = matching columns of J.
__device__ void jacobi_tail_1cta(const double* X, const double* J, int l, int k,
                                 double* __restrict__ Ub, int64_t ldu, double* __restrict__ s_out,
                                 double* __restrict__ Wk, int64_t ldw, double* gnorm, int* gperm,
                                 int* gsign) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kThreadsB = blockDim.x, kWarpsB = blockDim.x >> 5;
  // singular values = column norms
  for (int c = warp; c < l; c += kWarpsB) {
    double a = 0.0;
    for (int r = lane; r < l; r += 32) a += X[(int64_t)c * l + r] * X[(int64_t)c * l + r];
    a = warp_sum32(a);
    if (lane == 0) gnorm[c] = sqrt(a);
  }
  __syncthreads();
  // stable descending order: rank = #{i: s_i > s_j} + #{i < j: s_i == s_j}
  for (int j = tid; j < l; j += kThreadsB) {
    const double sj = gnorm[j];
    int rank = 0;
    for (int i = 0; i < l; ++i) {
      const double si = gnorm[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    gperm[rank] = j;
  }
  __syncthreads();
  // sign rule on U_B columns: largest |entry| positive, earliest row on ties
  for (int i = warp; i < l; i += kWarpsB) {
    const int c = gperm[i];
    double best = -1.0;
    int brow = 0;
    for (int r = lane; r < l; r += 32) {
      const double v = fabs(X[(int64_t)c * l + r]);
      if (v > best) {
        best = v;
        brow = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int orow = __shfl_xor_sync(0xffffffffu, brow, o);
      if (ob > best || (ob == best && orow < brow)) {
        best = ob;
        brow = orow;
      }
    }
    if (lane == 0) gsign[i] = (X[(int64_t)c * l + brow] < 0.0) ? -1 : 1;
  }
  __syncthreads();
  for (int i = tid; i < l; i += kThreadsB) s_out[i] = gnorm[gperm[i]];
  for (int r = warp; r < l; r += kWarpsB)
    for (int i = lane; i < l; i += 32) {
      const int c = gperm[i];
      const double sc = gnorm[c];
      const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
      Ub[(int64_t)r * ldu + i] = gsign[i] * X[(int64_t)c * l + r] * inv;
    }
  for (int r = warp; r < l; r += kWarpsB)
    for (int i = lane; i < k; i += 32) Wk[(int64_t)r * ldw + i] = gsign[i] * J[(int64_t)gperm[i] * l + r];
}

__global__ void __launch_bounds__(kThreads, 1)
    jacobi_kernel(const double* __restrict__ Rm, int64_t ldr, int l, int k, double* __restrict__ Ub,
                  int64_t ldu, double* __restrict__ s_out, double* __restrict__ Wk, int64_t ldw,
                  double* __restrict__ work, int* __restrict__ status, int j_in_smem, double tol,
                  int max_sweeps) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_rot;
  const int64_t ll = (int64_t)l * l;
  double* X = sm;
  double* J = j_in_smem ? sm + ll : work;
  // scratch after J in global: norms, perm, sign
  double* gnorm = work + ll;
  int* gperm = reinterpret_cast<int*>(gnorm + l);
  int* gsign = gperm + l;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = tid / kGroup, gl = tid % kGroup;
  for (int c = warp; c < l; c += kWarps)
    for (int r = lane; r < l; r += 32) {
      X[(int64_t)c * l + r] = Rm[(int64_t)c * ldr + r];
      J[(int64_t)c * l + r] = (r == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int L2 = l + (l & 1);
  const int npairs = L2 / 2;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < L2 - 1; ++round) {
      for (int pi = grp; pi < npairs; pi += kGroups) {
        const int pa = pi, pb = L2 - 1 - pi;  // circle method: position 0 fixed
        int p = pa == 0 ? 0 : 1 + (pa - 1 + round) % (L2 - 1);
        int q = 1 + (pb - 1 + round) % (L2 - 1);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= l) continue;  // dummy player when l is odd
        double* xp = X + (int64_t)p * l;
        double* xq = X + (int64_t)q * l;
        double a = 0.0, b = 0.0, g = 0.0;
        for (int r = gl; r < l; r += kGroup) {
          const double u = xp[r], v = xq[r];
          a = fma(u, u, a);
          b = fma(v, v, b);
          g = fma(u, v, g);
        }
        group_sum3(a, b, g);
        if (g != 0.0 && fabs(g) > tol * sqrt(a * b)) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t);
          const double sn = cs * t;
          for (int r = gl; r < l; r += kGroup) {
            const double u = xp[r], v = xq[r];
            xp[r] = cs * u - sn * v;
            xq[r] = sn * u + cs * v;
          }
          double* jp = J + (int64_t)p * l;
          double* jq = J + (int64_t)q * l;
          for (int r = gl; r < l; r += kGroup) {
            const double u = jp[r], v = jq[r];
            jp[r] = cs * u - sn * v;
            jq[r] = sn * u + cs * v;
          }
          if (gl == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    const int rotated = s_rot;
    __syncthreads();
    if (!rotated) break;
  }
  if (tid == 0) *status = (sweep >= max_sweeps) ? 1 : 0;
  jacobi_tail_1cta(X, J, l, k, Ub, ldu, s_out, Wk, ldw, gnorm, gperm, gsign);
}

// Single-CTA one-sided Jacobi with the pair's columns in REGISTERS
// (l <= 16 NR <= 128, X and J both in shared memory: 2 l^2 doubles <= 225 KB).
// Round-robin (circle) ordering: every round rotates the l/2 disjoint column
// pairs in parallel, one 16-lane group per pair; each lane loads its NR
// elements of x_p, x_q once, forms the three dot products, rotates in
// registers and stores once (then the same for J) — one shared-memory pass
// per column per round and one barrier per round.
template <int NR>
__global__ void __launch_bounds__(kThreads, 1)
    jacobi_rr_kernel(const double* __restrict__ Rm, int64_t ldr, int l, int k,
                     double* __restrict__ Ub, int64_t ldu, double* __restrict__ s_out,
                     double* __restrict__ Wk, int64_t ldw, double* __restrict__ work,
                     int* __restrict__ status, double tol, int max_sweeps) {
  extern __shared__ __align__(16) double sm[];
  const int64_t ll = (int64_t)l * l;
  double* X = sm;
  double* J = sm + ll;
  double* gnorm = work + ll;
  int* gperm = reinterpret_cast<int*>(gnorm + l);
  int* gsign = gperm + l;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = tid / kGroup, gl = tid % kGroup;
  for (int c = warp; c < l; c += kWarps)
    for (int r = lane; r < l; r += 32) {
      X[(int64_t)c * l + r] = Rm[(int64_t)c * ldr + r];
      J[(int64_t)c * l + r] = (r == c) ? 1.0 : 0.0;
    }
  __syncthreads();
  const int L2 = l + (l & 1);
  const int npairs = L2 / 2;
  const double tol2 = tol * tol;
  const unsigned hmask = (threadIdx.x & 16) ? 0xffff0000u : 0x0000ffffu;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    int rot = 0;
    // circle method (position 0 fixed): this group's players move one seat
    // per round, pp = 1 + (pa - 1 + round) mod (L2 - 1), kept incrementally
    const int pa = grp, pb = L2 - 1 - grp;
    int pp = pa, qq = pb;
    for (int round = 0; round < L2 - 1; ++round) {
      if (round > 0) {
        if (pa != 0 && ++pp == L2) pp = 1;
        if (++qq == L2) qq = 1;
      }
      if (grp < npairs) {
        int p = pp, q = qq;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q < l) {
          double* xp = X + (int64_t)p * l;
          double* xq = X + (int64_t)q * l;
          double u[NR], v[NR];
          double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
          for (int i = 0; i < NR; ++i) {
            const int r = gl + kGroup * i;
            u[i] = r < l ? xp[r] : 0.0;
            v[i] = r < l ? xq[r] : 0.0;
            a = fma(u[i], u[i], a);
            b = fma(v[i], v[i], b);
            g = fma(u[i], v[i], g);
          }
#pragma unroll
          for (int o = kGroup / 2; o > 0; o >>= 1) {
            a += __shfl_xor_sync(hmask, a, o);
            b += __shfl_xor_sync(hmask, b, o);
            g += __shfl_xor_sync(hmask, g, o);
          }
          if (g != 0.0 && g * g > tol2 * (a * b)) {
            const double zeta = (b - a) / (2.0 * g);
            const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
            const double cs = rsqrt(fma(t, t, 1.0));
            const double sn = cs * t;
#pragma unroll
            for (int i = 0; i < NR; ++i) {
              const int r = gl + kGroup * i;
              if (r < l) {
                xp[r] = cs * u[i] - sn * v[i];
                xq[r] = sn * u[i] + cs * v[i];
              }
            }
            double* jp = J + (int64_t)p * l;
            double* jq = J + (int64_t)q * l;
            // all loads of the two J columns before any store (no
            // load-store-load serialisation on possible aliasing)
            double ju[NR], jv[NR];
#pragma unroll
            for (int i = 0; i < NR; ++i) {
              const int r = gl + kGroup * i;
              ju[i] = r < l ? jp[r] : 0.0;
              jv[i] = r < l ? jq[r] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < NR; ++i) {
              const int r = gl + kGroup * i;
              if (r < l) {
                jp[r] = cs * ju[i] - sn * jv[i];
                jq[r] = sn * ju[i] + cs * jv[i];
              }
            }
            rot = 1;
          }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rot)) break;
  }
  if (tid == 0) {
    status[0] = (sweep >= max_sweeps) ? 1 : 0;
    status[1] = sweep;  // sweeps run (diagnostics, XB_TRACE)
  }
  jacobi_tail_1cta(X, J, l, k, Ub, ldu, s_out, Wk, ldw, gnorm, gperm, gsign);
}

// ---------------------------------------------------------------------------
// Cluster one-sided Jacobi (l <= 128): the single-CTA kernel above is bound by
// one SM's FP64 issue rate and its per-round latency chain (3.4 us per round
// at l = 120: 6 sweeps x 119 rounds = 2.4 ms). Here the l/2 column pairs of a
// round are spread over a thread-block cluster of kJC CTAs as a Brent-Luk
// systolic array: every CTA owns S consecutive SEATS (a top and a bottom
// column each, X and J side by side in its shared memory), one warp per seat.
// A round is: load the seat's two columns (local shared memory), the three dot
// products, the rotation in registers, then STORE the rotated columns straight
// into the seats they occupy next round — the neighbour's shared memory
// through DSMEM where the seat belongs to another CTA (two columns per CTA
// boundary per round) — into the other half of a ping-pong buffer, and one
// cluster barrier. Seat movement is the circle method: top[0] fixed,
// top[i] -> top[i+1], top[P-1] -> bottom[P-1], bottom[i] -> bottom[i-1],
// bottom[0] -> top[1]; after 2P-1 rounds every pair has met once and every
// column is back in its first seat. Column identities travel with the data
// so that the tail's stable sort sees the original column order.

// NR: doubles per lane per column (column length padded to 32 NR; a lane
// holds rows 2 lane + 64 i + {0, 1}: 16-byte shared-memory accesses).
//
// A sweep ends the iteration when none of its rotations was larger than
// thr = sqrt(tol / 4l): by the quadratic convergence of the method the
// off-diagonal cosines left behind are then O(l thr^2) <= tol, which is what
// the extra rotation-free sweep of the single-CTA kernels verifies — one
// sweep in seven at l = 120.
//
// Measured alternatives (profiles/r02_jacobi_cluster.md): seat-to-seat
// mbarriers instead of the cluster barrier (arrive.release.cluster per lane:
// slower; st.async + complete_tx: every byte crosses the cluster network,
// slower at l = 120, 10-20 % faster at l <= 64).
template <int NR>
__global__ void __launch_bounds__(256, 1)
    jacobi_cluster_kernel(const double* __restrict__ Rm, int64_t ldr, int l, int k,
                          double* __restrict__ Ub, int64_t ldu, double* __restrict__ s_out,
                          double* __restrict__ Wk, int64_t ldw, double* work,
                          int* __restrict__ status, double tol, int max_sweeps) {
  static_assert(NR % 2 == 0, "two doubles per access");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int LP = 32 * NR;  // padded column length; rows >= l stay zero
  constexpr int NV = NR / 2;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_id[2][2][8];
  __shared__ int s_rot[2];
  __shared__ int s_perm[128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster.block_rank();
  const int nc = (int)cluster.num_blocks();
  const int L2 = l + (l & 1), P = L2 / 2;
  const int S = (P + nc - 1) / nc;  // seats per CTA (<= 8 for l <= 128)
  const int seat = rank * S + warp;
  const bool active = warp < S && seat < P;
  // column slot (buffer, row 0 top / 1 bottom, local seat): X then J
  auto slot = [&](int buf, int row, int ls) -> double* {
    return sm + (int64_t)((buf * 2 + row) * S + ls) * (2 * LP);
  };
  const int64_t ll = (int64_t)l * l;
  double* Xg = work;  // final columns by original index (tail)
  double* Jg = work + ll;
  double* gnorm = work + 2 * ll;
  int* gsign = reinterpret_cast<int*>(gnorm + l);
  if (tid < 2) s_rot[tid] = 0;
  if (active) {
    // first seats: top[i] = column i, bottom[i] = column L2-1-i (the dummy
    // zero column of an odd l sits in bottom[0])
#pragma unroll
    for (int row = 0; row < 2; ++row) {
      const int c = row == 0 ? seat : L2 - 1 - seat;
      double* x = slot(0, row, warp);
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int r = lane + 32 * i;
        x[r] = (c < l && r < l) ? Rm[(int64_t)c * ldr + r] : 0.0;
        x[LP + r] = (c < l && r == c) ? 1.0 : 0.0;
      }
      if (lane == 0) s_id[0][row][warp] = c;
    }
  }
  // destination seats of this warp's two columns (fixed for the whole run)
  const int sseat = active ? seat : 0;
  int drow_t = 0, dseat_t = sseat, drow_b = 1, dseat_b = sseat;
  if (sseat > 0) {
    if (sseat < P - 1) dseat_t = sseat + 1;
    else drow_t = 1;  // top[P-1] -> bottom[P-1]
  }
  if (sseat > 0) {
    dseat_b = sseat - 1;
  } else if (P > 1) {  // bottom[0] -> top[1]
    drow_b = 0;
    dseat_b = 1;
  }
  const int drank_t = dseat_t / S, dls_t = dseat_t - drank_t * S;
  const int drank_b = dseat_b / S, dls_b = dseat_b - drank_b * S;
  // buffer 0's slots (buffer 1 lies a fixed stride further); seats of this
  // CTA are addressed as plain shared memory and only the two columns that
  // cross a CTA boundary go through DSMEM
  double* const dst_t = drank_t == rank ? slot(0, drow_t, dls_t)
                                        : cluster.map_shared_rank(slot(0, drow_t, dls_t), drank_t);
  double* const dst_b = drank_b == rank ? slot(0, drow_b, dls_b)
                                        : cluster.map_shared_rank(slot(0, drow_b, dls_b), drank_b);
  int* const did_t = drank_t == rank ? &s_id[0][drow_t][dls_t]
                                     : cluster.map_shared_rank(&s_id[0][drow_t][dls_t], drank_t);
  int* const did_b = drank_b == rank ? &s_id[0][drow_b][dls_b]
                                     : cluster.map_shared_rank(&s_id[0][drow_b][dls_b], drank_b);
  const int64_t bstride = (int64_t)2 * S * 2 * LP;  // doubles per buffer
  cluster.sync();
  const double tol2 = tol * tol;
  const double thr2 = fmax(tol2, tol / (4.0 * l));
  const int rounds = L2 - 1;
  int par = 0, sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    const int fs = sweep & 1;
    for (int round = 0; round < rounds; ++round) {
      if (active) {
        const double2* xt = reinterpret_cast<const double2*>(slot(par, 0, warp));
        const double2* xb = reinterpret_cast<const double2*>(slot(par, 1, warp));
        double2 u[NV], v[NV], ju[NV], jv[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          u[i] = xt[lane + 32 * i];
          v[i] = xb[lane + 32 * i];
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          ju[i] = xt[LP / 2 + lane + 32 * i];
          jv[i] = xb[LP / 2 + lane + 32 * i];
        }
        const int idt = s_id[par][0][warp], idb = s_id[par][1][warp];
        // two partial sums per dot product (FP64 latency, not rate, paces a round)
        double a = u[0].x * u[0].x, b = v[0].x * v[0].x, g = u[0].x * v[0].x;
        double a1 = u[0].y * u[0].y, b1 = v[0].y * v[0].y, g1 = u[0].y * v[0].y;
#pragma unroll
        for (int i = 1; i < NV; ++i) {
          a = fma(u[i].x, u[i].x, a);
          b = fma(v[i].x, v[i].x, b);
          g = fma(u[i].x, v[i].x, g);
          a1 = fma(u[i].y, u[i].y, a1);
          b1 = fma(v[i].y, v[i].y, b1);
          g1 = fma(u[i].y, v[i].y, g1);
        }
        a += a1;
        b += b1;
        g += g1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        const double gg = g * g, ab = a * b;
        if (g != 0.0 && gg > tol2 * ab) {
          // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = (b - a) / 2g,
          // written without the division: with d = b - a, h = 2g (both scaled
          // by a power of two so the squares stay in range),
          // den = |d| + sqrt(d^2 + h^2): cs = den / sqrt(den^2 + h^2),
          // sn = sign(d) sign(h) |h| / sqrt(den^2 + h^2)
          double d = b - a, h = 2.0 * g;
          const double mx = fmax(fabs(d), fabs(h));
          int ex = (__double2hiint(mx) >> 20) & 0x7ff;
          ex = ex < 1 ? 1 : (ex > 2045 ? 2045 : ex);
          const double sc = __hiloint2double((2046 - ex) << 20, 0);
          d *= sc;
          h *= sc;
          const double den = fabs(d) + sqrt(fma(d, d, h * h));
          const double w = rsqrt(fma(den, den, h * h));
          const double cs = den * w;
          const double sn =
              ((__double2hiint(d) ^ __double2hiint(h)) < 0) ? -fabs(h) * w : fabs(h) * w;
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            double2 nu, nv;
            nu.x = cs * u[i].x - sn * v[i].x;
            nu.y = cs * u[i].y - sn * v[i].y;
            nv.x = sn * u[i].x + cs * v[i].x;
            nv.y = sn * u[i].y + cs * v[i].y;
            u[i] = nu;
            v[i] = nv;
            nu.x = cs * ju[i].x - sn * jv[i].x;
            nu.y = cs * ju[i].y - sn * jv[i].y;
            nv.x = sn * ju[i].x + cs * jv[i].x;
            nv.y = sn * ju[i].y + cs * jv[i].y;
            ju[i] = nu;
            jv[i] = nv;
          }
          if (lane == 0 && gg > thr2 * ab) s_rot[fs] = 1;
        }
        double2* ot = reinterpret_cast<double2*>(dst_t + (par ^ 1) * bstride);
        double2* ob = reinterpret_cast<double2*>(dst_b + (par ^ 1) * bstride);
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          ot[lane + 32 * i] = u[i];
          ob[lane + 32 * i] = v[i];
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          ot[LP / 2 + lane + 32 * i] = ju[i];
          ob[LP / 2 + lane + 32 * i] = jv[i];
        }
        if (lane == 0) {
          did_t[(par ^ 1) * 16] = idt;
          did_b[(par ^ 1) * 16] = idb;
        }
      }
      cluster.sync();
      // every CTA read last sweep's flags before it arrived at this barrier
      if (round == 0 && tid == 0) s_rot[fs ^ 1] = 0;
      par ^= 1;
    }
    int any = 0;
    for (int r = 0; r < nc; ++r) any |= *cluster.map_shared_rank(&s_rot[fs], r);
    if (!any) break;
  }
  if (tid == 0 && rank == 0) {
    status[0] = (sweep >= max_sweeps) ? 1 : 0;
    status[1] = sweep;
  }
  // Tail. Norms, signs (largest |entry| positive, earliest row on ties,
  // kernels.py:556-561) and the columns themselves go to global scratch by
  // original column index; after a cluster barrier every CTA ranks the norms
  // (stable descending, kernels.py:535) and writes its share of U_B, s, W_k.
  if (active) {
#pragma unroll
    for (int row = 0; row < 2; ++row) {
      const int c = s_id[par][row][warp];
      if (c >= l) continue;
      const double* x = slot(par, row, warp);
      double a = 0.0, best = -1.0;
      int brow = 0;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        const int r = lane + 32 * i;
        const double xv = x[r];
        a = fma(xv, xv, a);
        if (r < l) {
          Xg[(int64_t)c * l + r] = xv;
          Jg[(int64_t)c * l + r] = x[LP + r];
          if (fabs(xv) > best) {
            best = fabs(xv);
            brow = r;
          }
        }
      }
      a = warp_sum32(a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orow = __shfl_xor_sync(0xffffffffu, brow, o);
        if (ob > best || (ob == best && orow < brow)) {
          best = ob;
          brow = orow;
        }
      }
      if (lane == 0) {
        gnorm[c] = sqrt(a);
        gsign[c] = (x[brow] < 0.0) ? -1 : 1;
      }
    }
  }
  __threadfence();
  cluster.sync();
  for (int j = tid; j < l; j += blockDim.x) {
    const double sj = gnorm[j];
    int rk = 0;
    for (int i = 0; i < l; ++i) {
      const double si = gnorm[i];
      rk += (si > sj) || (si == sj && i < j);
    }
    s_perm[rk] = j;
  }
  __syncthreads();
  const int nwarps = blockDim.x >> 5;
  for (int i = rank * nwarps + warp; i < l; i += nc * nwarps) {
    const int c = s_perm[i];
    const double scn = gnorm[c];
    const double inv = scn > 0.0 ? 1.0 / scn : 0.0;
    const int sg = gsign[c];
    if (lane == 0) s_out[i] = scn;
    for (int r = lane; r < l; r += 32) {
      Ub[(int64_t)r * ldu + i] = sg * Xg[(int64_t)c * l + r] * inv;
      if (i < k) Wk[(int64_t)r * ldw + i] = sg * Jg[(int64_t)c * l + r];
    }
  }
  // no CTA may exit while a neighbour can still address its shared memory
  cluster.sync();
}

// Shared tail of the cooperative Jacobi kernels: singular values = column
// norms of X, stable descending order, the sign rule of kernels.py:556-561,
// U_B = X[:, perm] / s (sign-fixed) and the first k columns of J.
__device__ void jacobi_finish_grid(const double* X, const double* J, int l, int k,
                                   double* __restrict__ Ub, int64_t ldu, double* __restrict__ s_out,
                                   double* __restrict__ Wk, int64_t ldw, double* gnorm, int* gperm,
                                   int* gsign) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t ll = (int64_t)l * l;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int gwarp = (int)(gtid >> 5);
  const int nwarps = (int)(gthreads >> 5);
  grid.sync();
  for (int c = gwarp; c < l; c += nwarps) {
    double a = 0.0;
    for (int r = lane; r < l; r += 32) a += X[(int64_t)c * l + r] * X[(int64_t)c * l + r];
    a = warp_sum32(a);
    if (lane == 0) gnorm[c] = sqrt(a);
  }
  grid.sync();
  for (int64_t j = gtid; j < l; j += gthreads) {
    const double sj = gnorm[j];
    int rank = 0;
    for (int i = 0; i < l; ++i) {
      const double si = gnorm[i];
      rank += (si > sj) || (si == sj && i < (int)j);
    }
    gperm[rank] = (int)j;
  }
  grid.sync();
  for (int i = gwarp; i < l; i += nwarps) {
    const int c = gperm[i];
    double best = -1.0;
    int brow = 0;
    for (int r = lane; r < l; r += 32) {
      const double v = fabs(X[(int64_t)c * l + r]);
      if (v > best) {
        best = v;
        brow = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int orow = __shfl_xor_sync(0xffffffffu, brow, o);
      if (ob > best || (ob == best && orow < brow)) {
        best = ob;
        brow = orow;
      }
    }
    if (lane == 0) gsign[i] = (X[(int64_t)c * l + brow] < 0.0) ? -1 : 1;
  }
  grid.sync();
  for (int64_t i = gtid; i < l; i += gthreads) s_out[i] = gnorm[gperm[i]];
  for (int64_t idx = gtid; idx < ll; idx += gthreads) {
    const int r = (int)(idx / l), i = (int)(idx - (int64_t)r * l);
    const int c = gperm[i];
    const double sc = gnorm[c];
    const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
    Ub[(int64_t)r * ldu + i] = gsign[i] * X[(int64_t)c * l + r] * inv;
  }
  for (int64_t idx = gtid; idx < (int64_t)l * k; idx += gthreads) {
    const int r = (int)(idx / k), i = (int)(idx - (int64_t)r * k);
    Wk[(int64_t)r * ldw + i] = gsign[i] * J[(int64_t)gperm[i] * l + r];
  }
}

// ---------------------------------------------------------------------------
// Cooperative multi-CTA Jacobi for large l (l x l does not fit one SM's
// shared memory: cfg4 l=220, cfg5 l=550). X and J live in global memory
// (L2-resident: 2 l^2 doubles), one warp per column pair, a grid-wide
// barrier between rounds. Same rotation, ordering, sort and sign rule as
// the single-CTA kernel.
__global__ void __launch_bounds__(256)
    jacobi_coop_kernel(const double* __restrict__ Rm, int64_t ldr, int l, int k,
                       double* __restrict__ Ub, int64_t ldu, double* __restrict__ s_out,
                       double* __restrict__ Wk, int64_t ldw, double* __restrict__ work,
                       int* __restrict__ status, double tol, int max_sweeps) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int64_t ll = (int64_t)l * l;
  double* X = work;
  double* J = work + ll;
  double* gnorm = work + 2 * ll;
  int* gperm = reinterpret_cast<int*>(gnorm + l);
  int* gsign = gperm + l;
  int* rotflag = gsign + l;  // max_sweeps ints, zeroed here
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int gwarp = (int)(gtid >> 5);
  const int nwarps = (int)(gthreads >> 5);
  for (int64_t idx = gtid; idx < ll; idx += gthreads) {
    const int c = (int)(idx / l), r = (int)(idx - (int64_t)c * l);
    X[idx] = Rm[(int64_t)c * ldr + r];
    J[idx] = (r == c) ? 1.0 : 0.0;
  }
  for (int64_t i = gtid; i < max_sweeps; i += gthreads) rotflag[i] = 0;
  grid.sync();
  const int L2 = l + (l & 1);
  const int npairs = L2 / 2;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int round = 0; round < L2 - 1; ++round) {
      for (int pi = gwarp; pi < npairs; pi += nwarps) {
        const int pa = pi, pb = L2 - 1 - pi;
        int p = pa == 0 ? 0 : 1 + (pa - 1 + round) % (L2 - 1);
        int q = 1 + (pb - 1 + round) % (L2 - 1);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q >= l) continue;
        double* xp = X + (int64_t)p * l;
        double* xq = X + (int64_t)q * l;
        double a = 0.0, b = 0.0, g = 0.0;
        // L2-coherent loads (__ldcg): columns move between SMs every round
        for (int r = lane; r < l; r += 32) {
          const double u = __ldcg(xp + r), v = __ldcg(xq + r);
          a = fma(u, u, a);
          b = fma(v, v, b);
          g = fma(u, v, g);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (g != 0.0 && fabs(g) > tol * sqrt(a * b)) {
          const double zeta = (b - a) / (2.0 * g);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t);
          const double sn = cs * t;
          double* jp = J + (int64_t)p * l;
          double* jq = J + (int64_t)q * l;
          for (int r = lane; r < l; r += 32) {
            const double u = __ldcg(xp + r), v = __ldcg(xq + r);
            __stcg(xp + r, cs * u - sn * v);
            __stcg(xq + r, sn * u + cs * v);
            const double uj = __ldcg(jp + r), vj = __ldcg(jq + r);
            __stcg(jp + r, cs * uj - sn * vj);
            __stcg(jq + r, sn * uj + cs * vj);
          }
          if (lane == 0) rotflag[sweep] = 1;
        }
      }
      grid.sync();
    }
    if (*(volatile int*)&rotflag[sweep] == 0) break;
  }
  if (gtid == 0) *status = (sweep >= max_sweeps) ? 1 : 0;
  jacobi_finish_grid(X, J, l, k, Ub, ldu, s_out, Wk, ldw, gnorm, gperm, gsign);
}

// ---------------------------------------------------------------------------
// Blocked one-sided Jacobi on a cooperative grid (replaces the column-pair
// cooperative kernel for every l that does not fit one CTA: cfg4 l=220,
// cfg5 l=550). Columns form nb blocks of `bs`; each outer round pairs blocks
// round-robin and one CTA takes a block pair: it loads the <= 2 bs columns of
// X and of J into shared memory, runs one inner cyclic sweep over all pairs
// of those columns (all 256 threads busy: 256 / bs lanes per pair) rotating
// both in place, and writes them back. Rounds per sweep drop from l - 1 (each a grid barrier with
// L2-latency-bound column traffic) to nb - 1. Convergence: a sweep in which
// no pair needed a rotation (|g| <= tol sqrt(a b)), as in the scalar kernels.
constexpr int kJT = 256;

template <int LANES>
__device__ __forceinline__ void lanes_sum3(double& a, double& b, double& c) {
  if constexpr (LANES == 16) {
    group_sum3(a, b, c);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
  }
}

template <int LANES>
__global__ void __launch_bounds__(kJT, 1)
    jacobi_block_kernel(const double* __restrict__ Rm, int64_t ldr, int l, int k,
                        double* __restrict__ Ub, int64_t ldu, double* __restrict__ s_out,
                        double* __restrict__ Wk, int64_t ldw, double* __restrict__ work,
                        int* __restrict__ status, double tol, int max_sweeps, int bs) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double smj[];
  const int64_t ll = (int64_t)l * l;
  double* X = work;
  double* J = work + ll;
  double* gnorm = work + 2 * ll;
  int* gperm = reinterpret_cast<int*>(gnorm + l);
  int* gsign = gperm + l;
  int* rotflag = gsign + l;
  const int W2 = 2 * bs;               // max columns per CTA
  double* xs = smj;                    // [W2][l] column-major: X[:, S]
  double* js = xs + (int64_t)W2 * l;   // [W2][l]: J[:, S]
  __shared__ int scol[64];
  __shared__ int s_rot, s_big;
  const double tol2 = tol * tol;
  const double thr2 = fmax(tol2, tol / (4.0 * l));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + tid;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = gtid; idx < ll; idx += gthreads) {
    const int c = (int)(idx / l), r = (int)(idx - (int64_t)c * l);
    X[idx] = Rm[(int64_t)c * ldr + r];
    J[idx] = (r == c) ? 1.0 : 0.0;
  }
  for (int64_t i = gtid; i < max_sweeps; i += gthreads) rotflag[i] = 0;
  grid.sync();
  const int nb = (l + bs - 1) / bs;
  const int NB2 = nb + (nb & 1);
  const int grp = tid / LANES, gl = tid % LANES;  // kJT / LANES pairs in flight
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int round = 0; round < NB2 - 1; ++round) {
      for (int pi = blockIdx.x; pi < NB2 / 2; pi += gridDim.x) {
        const int pa = pi, pb = NB2 - 1 - pi;
        const int bi = pa == 0 ? 0 : 1 + (pa - 1 + round) % (NB2 - 1);
        const int bj = 1 + (pb - 1 + round) % (NB2 - 1);
        // column set S = block bi (+ block bj unless it is the dummy)
        if (tid == 0) {
          int w = 0;
          for (int blk = 0; blk < 2; ++blk) {
            const int bb = blk == 0 ? min(bi, bj) : max(bi, bj);
            if (bb >= nb) continue;
            for (int c = bb * bs; c < min(l, (bb + 1) * bs); ++c) scol[w++] = c;
          }
          s_rot = 0;
          s_big = 0;
          scol[63] = w;
        }
        __syncthreads();
        const int w = scol[63];
        // global (L2) -> shared memory with cp.async: every element of the
        // <= 2 bs columns of X and J in flight at once (a load -> store loop
        // per column paid one L2 latency per 32 rows)
        for (int c = warp; c < w; c += kJT / 32) {
          const double* xg = X + (int64_t)scol[c] * l;
          const double* jg = J + (int64_t)scol[c] * l;
          const uint32_t xd = (uint32_t)__cvta_generic_to_shared(xs + (int64_t)c * l);
          const uint32_t jd = (uint32_t)__cvta_generic_to_shared(js + (int64_t)c * l);
          for (int r = lane; r < l; r += 32) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(xd + 8u * r), "l"(xg + r)
                         : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(jd + 8u * r), "l"(jg + r)
                         : "memory");
          }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        // one inner cyclic sweep over the w columns (circle ordering); the
        // rotations act on X[:, S] and J[:, S] in shared memory
        const int w2 = w + (w & 1);
        for (int ir = 0; ir < w2 - 1; ++ir) {
          for (int q0 = grp; q0 < w2 / 2; q0 += kJT / LANES) {
            const int qa = q0, qb = w2 - 1 - q0;
            int p = qa == 0 ? 0 : 1 + (qa - 1 + ir) % (w2 - 1);
            int q = 1 + (qb - 1 + ir) % (w2 - 1);
            if (p > q) {
              const int t = p;
              p = q;
              q = t;
            }
            if (q >= w) continue;
            double* xp = xs + (int64_t)p * l;
            double* xq = xs + (int64_t)q * l;
            // two independent accumulator sets: the loop is LDS-latency bound
            double a0 = 0.0, b0 = 0.0, g0 = 0.0, a1 = 0.0, b1 = 0.0, g1 = 0.0;
            int r = gl;
            for (; r + LANES < l; r += 2 * LANES) {
              const double u = xp[r], v = xq[r], u2 = xp[r + LANES], v2 = xq[r + LANES];
              a0 = fma(u, u, a0);
              b0 = fma(v, v, b0);
              g0 = fma(u, v, g0);
              a1 = fma(u2, u2, a1);
              b1 = fma(v2, v2, b1);
              g1 = fma(u2, v2, g1);
            }
            if (r < l) {
              const double u = xp[r], v = xq[r];
              a0 = fma(u, u, a0);
              b0 = fma(v, v, b0);
              g0 = fma(u, v, g0);
            }
            double a = a0 + a1, b = b0 + b1, g = g0 + g1;
            lanes_sum3<LANES>(a, b, g);
            const double gg = g * g, ab = a * b;
            if (g != 0.0 && gg > tol2 * ab) {
              // rotation without the FP64 divisions (as jacobi_cluster_kernel):
              // d = b - a, h = 2g scaled by a power of two, den = |d| + sqrt(d^2 + h^2),
              // cs = den / sqrt(den^2 + h^2), sn = sign(d) sign(h) |h| / sqrt(den^2 + h^2)
              double d = b - a, h = 2.0 * g;
              const double mx = fmax(fabs(d), fabs(h));
              int ex = (__double2hiint(mx) >> 20) & 0x7ff;
              ex = ex < 1 ? 1 : (ex > 2045 ? 2045 : ex);
              const double sc = __hiloint2double((2046 - ex) << 20, 0);
              d *= sc;
              h *= sc;
              const double den = fabs(d) + sqrt(fma(d, d, h * h));
              const double wr = rsqrt(fma(den, den, h * h));
              const double cs = den * wr;
              const double sn =
                  ((__double2hiint(d) ^ __double2hiint(h)) < 0) ? -fabs(h) * wr : fabs(h) * wr;
              double* jp = js + (int64_t)p * l;
              double* jq = js + (int64_t)q * l;
              // four rows per pass, every load before the first store (a
              // load -> fma -> store loop is a chain of dependent latencies)
              int rr = gl;
              for (; rr + 3 * LANES < l; rr += 4 * LANES) {
                double u[4], v[4], uj[4], vj[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  u[i] = xp[rr + i * LANES];
                  v[i] = xq[rr + i * LANES];
                  uj[i] = jp[rr + i * LANES];
                  vj[i] = jq[rr + i * LANES];
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  xp[rr + i * LANES] = cs * u[i] - sn * v[i];
                  xq[rr + i * LANES] = sn * u[i] + cs * v[i];
                  jp[rr + i * LANES] = cs * uj[i] - sn * vj[i];
                  jq[rr + i * LANES] = sn * uj[i] + cs * vj[i];
                }
              }
              for (; rr < l; rr += LANES) {
                const double u = xp[rr], v = xq[rr];
                const double uj = jp[rr], vj = jq[rr];
                xp[rr] = cs * u - sn * v;
                xq[rr] = sn * u + cs * v;
                jp[rr] = cs * uj - sn * vj;
                jq[rr] = sn * uj + cs * vj;
              }
              // only rotations above thr keep the iteration going (a sweep of
              // tiny rotations leaves <= tol behind: no rotation-free check sweep)
              if (gl == 0) {
                s_rot = 1;
                if (gg > thr2 * ab) s_big = 1;
              }
            }
          }
          __syncthreads();
        }
        if (s_rot) {
          for (int c = warp; c < w; c += kJT / 32) {
            double* xg = X + (int64_t)scol[c] * l;
            double* jg = J + (int64_t)scol[c] * l;
            const double* xd = xs + (int64_t)c * l;
            const double* jd = js + (int64_t)c * l;
            for (int r = lane; r < l; r += 32) {
              __stcg(xg + r, xd[r]);
              __stcg(jg + r, jd[r]);
            }
          }
          if (tid == 0 && s_big) rotflag[sweep] = 1;
        }
        __syncthreads();
      }
      grid.sync();
    }
    if (*(volatile int*)&rotflag[sweep] == 0) break;
  }
  if (gtid == 0) *status = (sweep >= max_sweeps) ? 1 : 0;
  jacobi_finish_grid(X, J, l, k, Ub, ldu, s_out, Wk, ldw, gnorm, gperm, gsign);
}

}  // namespace

size_t chol_work_doubles(int l) {
  const size_t nb = (size_t)(l + kCB - 1) / kCB, lp = nb * kCB;
  return std::max(2 * lp * lp + nb * kCB * kCB, (size_t)l * l);
}

void launch_chol_inv(const double* G, int64_t ldg, int l, double tau, double* R, double* Rinv,
                     int64_t ldr, int* flag, double* ws_in, cudaStream_t st) {
  XB_REQUIRE(l <= 4096, XB_EUNSUPPORTED, "chol_inv: l > 4096");
  const size_t bytes = (size_t)l * (l | 1) * sizeof(double);
  // XB_CHOL=coop forces the cooperative version (tests), =single the 1-CTA one
  static const int mode = [] {
    const char* e = knob("XB_CHOL");
    return e ? (strcmp(e, "coop") == 0 ? 1 : (strcmp(e, "single") == 0 ? 2 : 0)) : 0;
  }();
  const int use_smem = bytes + 26 * 1024 <= max_dyn_smem();
  if (mode == 1 || (mode == 0 && !use_smem) || l > 1024) {
    double* ws = ws_in;
    if (!ws)
      XB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), chol_work_doubles(l) * sizeof(double), st));
    int per_sm = 0;
    XB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chol_coop_kernel, kCT, 0));
    const int blocks = std::max(1, std::min(kNumSMs, kNumSMs * per_sm));
    void* args[] = {(void*)&G, (void*)&ldg, (void*)&l, (void*)&tau, (void*)&R,
                    (void*)&Rinv, (void*)&ldr, (void*)&flag, (void*)&ws};
    XB_CUDA(cudaLaunchCooperativeKernel((void*)chol_coop_kernel, dim3(blocks), dim3(kCT), args, 0, st));
    check_launch("chol_coop");
    if (!ws_in) XB_CUDA(cudaFreeAsync(ws, st));
    return;
  }
  static const bool blocked = [] {
    const char* e = knob("XB_CHOL_BLOCKED");
    return !(e && atoi(e) == 0);
  }();
  if (use_smem && blocked && l <= 256) {
    XB_CUDA(cudaFuncSetAttribute(chol_inv_blocked_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    chol_inv_blocked_kernel<<<1, kThreads, bytes, st>>>(G, ldg, l, tau, R, Rinv, ldr, flag);
    check_launch("chol_inv");
    return;
  }
  double* gw = use_smem ? nullptr : ws_in;
  const bool own = !use_smem && !gw;
  if (own) XB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&gw), bytes, st));
  const size_t dyn = use_smem ? bytes : 0;
  XB_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)dyn));
  chol_inv_kernel<<<1, kThreads, dyn, st>>>(G, ldg, l, tau, R, Rinv, ldr, flag, gw, use_smem);
  check_launch("chol_inv");
  if (own) XB_CUDA(cudaFreeAsync(gw, st));
}

constexpr int kMaxSweeps = 60;

size_t jacobi_work_doubles(int l) {
  return 2 * (size_t)l * l + 3 * (size_t)l + kMaxSweeps + 16;
}

void launch_jacobi_svd(const double* R, int64_t ldr, int l, int k, double* Ub, int64_t ldu,
                       double* s, double* Wk, int64_t ldw, double* work, int* status,
                       cudaStream_t st, double tol_req) {
  const size_t lim = max_dyn_smem() - 512;  // static: s_rot
  const size_t one = (size_t)l * l * sizeof(double);
  const double tol = tol_req > 0.0 ? tol_req : fmax(1e-15, (double)l * DBL_EPSILON);
  // one CTA while M's columns fit in shared memory, else (or on request,
  // XB_JACOBI=coop) the cooperative grid version
  static const int mode = [] {
    const char* e = knob("XB_JACOBI");
    return e ? (strcmp(e, "coop") == 0 ? 1
                : strcmp(e, "single") == 0 ? 2
                : strcmp(e, "pairs") == 0 ? 3
                : strcmp(e, "rr") == 0 ? 4
                : strcmp(e, "cluster") == 0 ? 5 : 0)
             : 0;
  }();
  // blocked cooperative kernel from l > 64 (l = 120: 3.3 ms vs 5.4 ms for
  // the single-CTA kernel), single CTA below
  // cluster kernel (one warp per column pair, seats spread over the CTAs of
  // one cluster: 16 where the device schedules such a cluster, else 8) for
  // 32 < l <= 128
  if ((mode == 0 || mode == 5) && l <= 128 && (l > 32 || mode == 5)) {
    static const int jnc_knob = [] {
      const char* e = knob("XB_JACOBI_NC");
      return e ? atoi(e) : 0;
    }();
    auto launch = [&](auto kern, int nr) {
      auto cfg_for = [&](int nc, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at) {
        const int P = (l + (l & 1)) / 2, S = (P + nc - 1) / nc;
        cfg = cudaLaunchConfig_t{};
        cfg.gridDim = dim3(nc);
        cfg.blockDim = dim3(32 * std::max(1, std::min(8, S)));
        cfg.dynamicSmemBytes = (size_t)2 * 2 * S * 2 * (32 * nr) * sizeof(double);
        cfg.stream = st;
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = nc;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
      };
      cudaLaunchConfig_t cfg;
      cudaLaunchAttribute at[1];
      XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      // a 16-CTA cluster (one warp per SM sub-partition at l = 120) needs the
      // opt-in attribute and a GPC with 16 free SMs: asked once per kernel
      static std::atomic<int> nc_cache[2];
      int nc = nc_cache[nr == 4].load();
      if (nc == 0) {
        nc = 8;
        if (jnc_knob != 8 &&
            cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                cudaSuccess) {
          cfg_for(16, cfg, at);
          int n = 0;
          if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n >= 1) nc = 16;
        }
        cudaGetLastError();
        nc_cache[nr == 4].store(nc);
      }
      cfg_for(nc, cfg, at);
      cudaError_t le = cudaLaunchKernelEx(&cfg, kern, R, ldr, l, k, Ub, ldu, s, Wk, ldw, work,
                                          status, tol, (int)kMaxSweeps);
      if (le != cudaSuccess && nc == 16) {
        // the 16-CTA cluster could not be placed after all: the portable size
        cudaGetLastError();
        nc_cache[nr == 4].store(8);
        cfg_for(8, cfg, at);
        le = cudaLaunchKernelEx(&cfg, kern, R, ldr, l, k, Ub, ldu, s, Wk, ldw, work, status, tol,
                                (int)kMaxSweeps);
      }
      XB_CUDA(le);
    };
    if (l <= 64) launch(jacobi_cluster_kernel<2>, 2);
    else launch(jacobi_cluster_kernel<4>, 4);
    check_launch("jacobi_cluster");
    if (getenv("XB_TRACE")) {
      int hs[2] = {0, 0};
      XB_CUDA(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
      XB_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr, "[xb] jacobi_cluster l=%d: %d sweeps\n", l, hs[1]);
    }
    return;
  }
  // register single-CTA kernel while X and J fit in shared memory (l <= 128)
  if ((mode == 0 || mode == 4) && l <= 128 && 2 * one <= lim) {
    const int dyn = (int)(2 * one);
#define XB_JRR(NR)                                                                            \
  do {                                                                                        \
    XB_CUDA(cudaFuncSetAttribute(jacobi_rr_kernel<NR>,                                        \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));          \
    jacobi_rr_kernel<NR><<<1, kThreads, dyn, st>>>(R, ldr, l, k, Ub, ldu, s, Wk, ldw, work,   \
                                                   status, tol, kMaxSweeps);                  \
  } while (0)
    if (l <= 32) XB_JRR(2);
    else if (l <= 64) XB_JRR(4);
    else XB_JRR(8);
#undef XB_JRR
    check_launch("jacobi_rr");
    if (getenv("XB_TRACE")) {
      int hs[2] = {0, 0};
      XB_CUDA(cudaMemcpyAsync(hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
      XB_CUDA(cudaStreamSynchronize(st));
      fprintf(stderr, "[xb] jacobi_rr l=%d: %d sweeps\n", l, hs[1]);
    }
    return;
  }
  const bool coop = mode == 1 || mode == 3 || (mode == 0 && (one > lim || l > 64));
  if (coop) {
    int max_sweeps = kMaxSweeps;
    if (mode != 3) {
      // blocked: bs columns per block (XB_JACOBI_BS, default 4: l = 552 ran
      // 28.9 ms at bs 4, 33 ms at 8, 68 ms at 16; l = 120 3.3 ms), halved until
      // the 2 bs columns of a block pair fit in shared memory
      static const int bs0 = [] {
        const char* e = knob("XB_JACOBI_BS");
        return e ? std::max(2, std::min(16, atoi(e))) : 4;
      }();
      int bs = bs0;
      auto need = [&](int b) { return (size_t)2 * (2 * b) * l * sizeof(double); };
      while (bs > 2 && need(bs) > lim) bs /= 2;
      XB_REQUIRE(need(bs) <= lim, XB_EUNSUPPORTED, "jacobi: l too large for the blocked kernel");
      const int dyn = (int)need(bs);
      // lanes per column pair: all 256 threads busy on the bs pairs of an inner round
      const bool l32 = kJT / bs >= 32;
      void* kern = l32 ? (void*)jacobi_block_kernel<32> : (void*)jacobi_block_kernel<16>;
      XB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
      const int nb = (l + bs - 1) / bs;
      const int blocks = std::max(1, std::min((nb + 1) / 2, kNumSMs));
      void* args[] = {(void*)&R,  (void*)&ldr, (void*)&l,      (void*)&k,   (void*)&Ub,
                      (void*)&ldu, (void*)&s,  (void*)&Wk,     (void*)&ldw, (void*)&work,
                      (void*)&status, (void*)&tol, (void*)&max_sweeps, (void*)&bs};
      XB_CUDA(cudaLaunchCooperativeKernel(kern, dim3(blocks), dim3(kJT), args, dyn, st));
      if (getenv("XB_TRACE")) {
        XB_CUDA(cudaStreamSynchronize(st));
        std::vector<int> rf(max_sweeps);
        XB_CUDA(cudaMemcpy(rf.data(), reinterpret_cast<int*>(work + 2 * (int64_t)l * l + l) + 2 * l,
                           max_sweeps * sizeof(int), cudaMemcpyDeviceToHost));
        int sw = 0;
        while (sw < max_sweeps && rf[sw]) ++sw;
        fprintf(stderr, "[xb] jacobi_block l=%d bs=%d: %d sweeps with rotations\n", l, bs, sw);
      }
      check_launch("jacobi_block");
      return;
    }
    int dev = 0, per_sm = 0;
    XB_CUDA(cudaGetDevice(&dev));
    XB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_coop_kernel, 256, 0));
    const int npairs = (l + (l & 1)) / 2;
    int blocks = std::max(1, std::min((npairs + 7) / 8, kNumSMs * std::max(per_sm, 1)));
    blocks = std::min(blocks, kNumSMs);
    void* args[] = {(void*)&R, (void*)&ldr, (void*)&l, (void*)&k, (void*)&Ub, (void*)&ldu,
                    (void*)&s, (void*)&Wk, (void*)&ldw, (void*)&work, (void*)&status,
                    (void*)&tol, (void*)&max_sweeps};
    XB_CUDA(cudaLaunchCooperativeKernel((void*)jacobi_coop_kernel, dim3(blocks), dim3(256), args, 0,
                                        st));
    check_launch("jacobi_coop");
    return;
  }
  const int j_in_smem = 2 * one <= lim;
  const size_t dyn = j_in_smem ? 2 * one : one;
  XB_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)dyn));
  jacobi_kernel<<<1, kThreads, dyn, st>>>(R, ldr, l, k, Ub, ldu, s, Wk, ldw, work, status,
                                          j_in_smem, tol, kMaxSweeps);
  check_launch("jacobi_svd");
}

}  // namespace xb
