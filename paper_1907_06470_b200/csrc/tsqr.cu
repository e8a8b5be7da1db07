// TSQR: the tall-skinny Householder QR as a reduction tree — the
// orthonormaliser that takes over when a CholQR Gram is not numerically
// positive definite (rank-deficient or very ill-conditioned sketches).
//
// The reference's thin_qr (kernels.py:297-351) is itself a flat tree: panels
// of max(r, 256) rows, each stacked under the running R and re-factored by
// Householder (_house / _householder_qr / _apply_reflectors, kernels.py:
// 247-294), then Q rebuilt backwards through the stashed reflectors. Here the
// same reflector convention (v[0] = 1, R_jj = +||x|| >= 0) runs as a G-ary
// tree so every SM works:
//
//   level 0   the rows split into blocks of <= rmax rows; each CTA factors
//             its block by blocked Householder (panels of NB columns: the
//             panel in shared memory, compact-WY T factor, trailing update
//             A -= V T^T V^T A by warps over 32-column chunks) and writes its
//             l x l R into the stack of level 1;
//   level L   groups of G = rmax / l stacked R factors, factored the same way,
//             until one block is left: its R is the QR's R;
//   Q         top-down: the root's reflectors applied to [I; 0], each block's
//             l x l slice of its parent's Q placed on top of zeros and
//             multiplied by the block's reflectors (right to left, panel by
//             panel E -= V T V^T E), level 0 writing Q itself.
//
// Both passes are ONE cooperative kernel each (grid.sync() between levels),
// and both return immediately when the Cholesky flag is 0, so the fallback
// costs two empty launches on the fast path. All sums run in a fixed order:
// results are bitwise reproducible.
//
// Row-sharded sketches: each rank factors its rows to a local
// l x l R, the ranks' R factors are all-gathered (world*l x l), every rank
// factors that stack identically (the root), forms its l x l slice of the
// root's Q and finishes its local Q top-down — the "R-factor gather" of the
// north star.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <vector>

#include "common.cuh"

namespace xb {
namespace {

namespace cg = cooperative_groups;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLevels = 40;
constexpr int kRound = 128;


struct Level {
  double* M;        // level matrix: rows x l, row-major, ld = Plan::ldm
  double* T;        // compact-WY factors: nblk x npan x NB x NB
  int64_t units;    // rows (level 0) or stacked R factors (levels >= 1)
  int64_t usize;    // rows per unit: 1 or l
  int64_t nblk;
};

struct Plan {
  int l, nb, npan, levels, rmax;
  int ldm;          // row stride of the level matrices: l rounded up to even (16-byte rows)
  int64_t rows;
  Level lv[kMaxLevels];
  double* Qb[2];    // Q of levels >= 1 (ping-pong), ld = ldm
};

__device__ __forceinline__ void block_rows(const Level& L, int64_t q, int64_t& s, int64_t& e) {
  s = q * L.units / L.nblk * L.usize;
  e = (q + 1) * L.units / L.nblk * L.usize;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int NB>
struct Smem {
  double* Ps;    // NB x rs panel, column-major (explicit V after factoring)
  double* part;  // NB x 256 stride, 128 used: W / W2 of a column round; Gram partials
  double* red;   // kWarps x NB
  double* tot;   // NB
  double* yjj;   // NB
  double* Gm;    // NB x NB
  double* Ts;    // NB x NB
  int rs;
};

template <int NB>
__device__ Smem<NB> carve(double* base, int rmax) {
  Smem<NB> s;
  s.rs = rmax + 1;
  s.Ps = base;
  s.part = s.Ps + (size_t)NB * s.rs;
  s.red = s.part + NB * 256;
  s.tot = s.red + kWarps * NB;
  s.yjj = s.tot + NB;
  s.Gm = s.yjj + NB;
  s.Ts = s.Gm + NB * NB;
  return s;
}

template <int NB>
constexpr size_t smem_doubles(int rmax) {
  return (size_t)NB * (rmax + 1) + NB * 256 + kWarps * NB + 2 * NB + 2 * NB * NB;
}



// Load panel columns [p0, p0 + nbc) of rows [p0, r) of A (row-major, lda)
// into Ps (column-major); columns nbc..NB-1 are zero. Eight loads per thread
// in flight (the block lives in L2; latency, not bandwidth, bounds this).
template <int NB>
__device__ void load_panel(const Smem<NB>& S, const double* A, int64_t lda, int64_t p0, int64_t r,
                           int nbc) {
  const int64_t rr = r - p0, total = rr * NB;
  for (int64_t base = threadIdx.x; base < total; base += 8 * kThreads) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t idx = base + (int64_t)u * kThreads;
      const int64_t i = idx / NB;
      const int k = (int)(idx - i * NB);
      v[u] = (idx < total && k < nbc) ? A[(p0 + i) * lda + p0 + k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t idx = base + (int64_t)u * kThreads;
      const int64_t i = idx / NB;
      const int k = (int)(idx - i * NB);
      if (idx < total) S.Ps[(size_t)k * S.rs + i] = v[u];
    }
  }
}

// Householder factorisation of the panel in shared memory (the reference's
// _house convention: v[0] = 1, beta, R_jj = mu >= 0). Leaves V below the
// diagonal, R on and above it, and the betas on Ts's diagonal. Four warps
// (one per scheduler) do it — the panel is a few hundred rows and per-column
// latency, not arithmetic, bounds it; the rest of the CTA waits at the
// closing barrier. Each of the PT threads owns the rows i = tid (mod PT) for
// all columns, so the update of column jj and the partial sums of column
// jj + 1 touch only the thread's own rows: two named barriers per column.
constexpr int kPanelThreads = 256;
__device__ __forceinline__ void panel_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(kPanelThreads) : "memory"); }

template <int NB>
__device__ void factor_panel(const Smem<NB>& S, int64_t rr, int nbc) {
  // Columns past nbc are zero in Ps: their reflectors come out as beta = 0
  // (identity) and leave every other column untouched, so all NB columns are
  // processed with compile-time column indices (no per-entry predicates).
  (void)nbc;
  constexpr int PT = kPanelThreads, PW = PT / 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < PT) {
#pragma unroll
    for (int jj = 0; jj < NB; ++jj) {
      double acc[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) acc[c] = 0.0;
      const double* xcol = S.Ps + (size_t)jj * S.rs;
      for (int64_t i = tid; i < rr; i += PT) {
        if (i <= jj) continue;  // own rows strictly below the diagonal row jj
        const double x = xcol[i];
        acc[jj] = fma(x, x, acc[jj]);
#pragma unroll
        for (int c = jj + 1; c < NB; ++c) acc[c] = fma(x, S.Ps[(size_t)c * S.rs + i], acc[c]);
      }
      // the butterflies level by level (independent shuffles in flight)
      __syncwarp();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = jj; c < NB; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
      if (lane == 0)
#pragma unroll
        for (int c = jj; c < NB; ++c) S.red[warp * NB + c] = acc[c];
      panel_bar();
      if (tid >= jj && tid < NB) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < PW; ++w) t += S.red[w * NB + tid];
        S.tot[tid] = t;
        S.yjj[tid] = S.Ps[(size_t)tid * S.rs + jj];
      }
      panel_bar();
      const double sigma = S.tot[jj], x0 = S.yjj[jj];
      double v0 = 1.0, beta, mu;
      if (sigma == 0.0) {
        beta = (x0 >= 0.0) ? 0.0 : 2.0;
        mu = (x0 >= 0.0) ? x0 : -x0;
      } else {
        mu = sqrt(x0 * x0 + sigma);
        v0 = (x0 <= 0.0) ? (x0 - mu) : (-sigma / (x0 + mu));
        beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
      }
      const double iv = sigma != 0.0 ? 1.0 / v0 : 0.0;
      double bw[NB];  // beta * w_c
#pragma unroll
      for (int c = jj + 1; c < NB; ++c) bw[c] = beta * (S.yjj[c] + S.tot[c] * iv);
      double* xc = S.Ps + (size_t)jj * S.rs;
      for (int64_t i = tid; i < rr; i += PT) {
        if (i <= jj) continue;
        // the row's panel entries in registers first: separate loads,
        // updates and stores (a load-update-store per entry serialises on
        // possible aliasing)
        double y[NB];
#pragma unroll
        for (int c = jj + 1; c < NB; ++c) y[c] = S.Ps[(size_t)c * S.rs + i];
        const double v = xc[i] * iv;
        xc[i] = v;
#pragma unroll
        for (int c = jj + 1; c < NB; ++c) S.Ps[(size_t)c * S.rs + i] = y[c] - bw[c] * v;
      }
      if (tid == jj) {  // the owner of row jj (jj < NB <= PT): R row jj
        xc[jj] = mu;
#pragma unroll
        for (int c = jj + 1; c < NB; ++c) S.Ps[(size_t)c * S.rs + jj] = S.yjj[c] - bw[c];
        S.Ts[jj * NB + jj] = beta;
      }
    }
  }
  __syncthreads();
}

// Ps -> explicit V (zeros above the diagonal, ones on it; zero columns past
// nbc), then T of H_0 ... H_{nbc-1} = I - V T V^T (Ts, upper triangular) from
// the betas on Ts's diagonal and the Gram of V.
template <int NB>
__device__ void build_T(const Smem<NB>& S, int64_t rr, int nbc, bool betas_in_T) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < NB * NB; idx += kThreads) {
    const int k = idx / NB, i = idx - k * NB;  // column k, row i < NB
    if (i < rr) {
      double& p = S.Ps[(size_t)k * S.rs + i];
      if (k >= nbc || i < k) p = 0.0;
      else if (i == k) p = 1.0;
    }
  }
  if (!betas_in_T) return;
  __syncthreads();
  // Gram G = V^T V on the FP64 tensor pipe: 8 x 8 tiles, rows split over warps
  constexpr int MT = (NB + 7) / 8, TILES = MT * MT, KSPL = kWarps / TILES;
  const int g = lane >> 2, t = lane & 3;
  if (warp < TILES * KSPL) {
    const int tile = warp % TILES, ks = warp / TILES;
    const int at = tile / MT, bt = tile % MT;
    const int ka = at * 8 + g, kb = bt * 8 + g;
    const int64_t i0 = ks * rr / KSPL, i1 = (ks + 1) * rr / KSPL;
    double c0 = 0.0, c1 = 0.0;
    for (int64_t i = i0; i < i1; i += 4) {
      const int64_t row = i + t;
      const bool ok = row < i1;
      const double a = (ok && ka < NB) ? S.Ps[(size_t)ka * S.rs + row] : 0.0;
      const double b = (ok && kb < NB) ? S.Ps[(size_t)kb * S.rs + row] : 0.0;
      dmma(c0, c1, a, b);
    }
    const int col = bt * 8 + 2 * t;
    if (ka < NB) {
      if (col < NB) S.part[ks * NB * NB + ka * NB + col] = c0;
      if (col + 1 < NB) S.part[ks * NB * NB + ka * NB + col + 1] = c1;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < NB * NB; idx += kThreads) {
    double v = 0.0;
    for (int ks = 0; ks < KSPL; ++ks) v += S.part[ks * NB * NB + idx];
    S.Gm[idx] = v;
  }
  __syncthreads();
  // T (upper triangular) by the recurrence T[0:j, j] = -beta_j T[0:j, 0:j] G[0:j, j];
  // lane i keeps row i of T in registers
  if (warp == 0) {
    double Tr[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) Tr[k] = (k == lane && k < nbc) ? S.Ts[k * NB + k] : 0.0;
#pragma unroll
    for (int j = 1; j < NB; ++j) {
      if (j < nbc) {
        const double bj = S.Ts[j * NB + j];
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < j; ++k)
          if (k >= lane) acc = fma(Tr[k], S.Gm[k * NB + j], acc);
        if (lane < j) Tr[j] = -bj * acc;
      }
    }
    __syncwarp();
    if (lane < NB)
#pragma unroll
      for (int k = 0; k < NB; ++k) S.Ts[lane * NB + k] = Tr[k];
  }
  __syncthreads();
}


// A[p0:r, cbeg:cend] -= V op(T) V^T A[p0:r, cbeg:cend]  (op = T^T when
// `transT`: the factorisation's Q^T update; op = T: the Q build). V, T in
// shared memory; both products on the FP64 tensor pipe (mma.sync m8n8k4:
// one instruction per 256 multiply-adds, where scalar FMAs spent most of the
// issue slots on operand traffic). Columns in rounds of 128:
//   W = V^T A   warps own (8-row k-tile of V^T, 32-column group) over a row
//               range; rows in batches of 16 (four k-steps into a fresh
//               accumulator, then folded into the running sum: shorter
//               rounding chains), operands straight from L2 into fragments;
//   W2 = op(T) W  one thread per column;
//   A -= V W2   warps own (8-row tile, 64-column group), C fragments loaded
//               from and stored back to A.
// (Measured alternatives, 1e6 x 120: staging A through a shared-memory ring
// by cp.async or 1-D bulk copies, 512-thread CTAs, one- and four-warp panel
// factorisations — all slower than this at 2 CTAs per SM.)
template <int NB, bool transT>
__device__ void apply_wy(const Smem<NB>& S, double* A, int64_t lda, int64_t p0, int64_t r,
                         int cbeg, int cend) {
  constexpr int MT = (NB + 7) / 8;  // k-tiles of V^T (8 rows each)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t rr = r - p0;
  double* Ab = A + p0 * lda;
  for (int c0 = cbeg; c0 < cend; c0 += kRound) {
    const int nc = min(kRound, cend - c0);
    // ---- W = V^T A  (NB x nc) -> S.part[k * 256 + col]
    const int ngrp = (nc + 31) >> 5;
    const int items = MT * ngrp;
    const int KH = items * 2 <= kWarps ? 2 : 1;  // row halves per item (partials -> part)
    for (int it2 = warp; it2 < items * KH; it2 += kWarps) {
      const int item = it2 % items, half = it2 / items;
      const int mt = item % MT, grp = item / MT;
      const int64_t ibeg = half * rr / KH, iend = (half + 1) * rr / KH;
      const int kv = mt * 8 + g;  // this lane's row of V^T in the A fragment
      const double* vrow = S.Ps + (size_t)(kv < NB ? kv : 0) * S.rs;
      int col[4];
      bool cok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        col[j] = grp * 32 + j * 8 + g;
        cok[j] = col[j] < nc;
      }
      double acc[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
      for (int64_t i = ibeg; i < iend; i += 16) {
        double bf[4][4], af[4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int64_t row = i + ks * 4 + t;
          const bool rok = row < iend;
          af[ks] = (rok && kv < NB) ? vrow[row] : 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) bf[ks][j] = (rok && cok[j]) ? Ab[row * lda + c0 + col[j]] : 0.0;
        }
        double p[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) p[j][0] = p[j][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(p[j][0], p[j][1], af[ks], bf[ks][j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[j][0] += p[j][0];
          acc[j][1] += p[j][1];
        }
      }
      // C fragment: row g of the k-tile, columns 2t, 2t + 1 of each n-tile
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cb = grp * 32 + j * 8 + 2 * t;
        if (kv < NB) {
          if (cb < nc) S.part[kv * 256 + half * 128 + cb] = acc[j][0];
          if (cb + 1 < nc) S.part[kv * 256 + half * 128 + cb + 1] = acc[j][1];
        }
      }
    }
    __syncthreads();
    // ---- W2 = op(T) W, one thread per column (negated: A += V (-W2))
    if (tid < nc) {
      double w[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k)
        w[k] = KH == 2 ? S.part[k * 256 + tid] + S.part[k * 256 + 128 + tid] : S.part[k * 256 + tid];
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        double u = 0.0;
        if (transT) {
#pragma unroll
          for (int j = 0; j <= k; ++j) u = fma(S.Ts[j * NB + k], w[j], u);
        } else {
#pragma unroll
          for (int j = k; j < NB; ++j) u = fma(S.Ts[k * NB + j], w[j], u);
        }
        S.part[k * 256 + tid] = -u;
      }
    }
    __syncthreads();
    // ---- A += V (-W2): tiles of 8 rows x 64 columns
    constexpr int KS = (NB + 3) / 4;  // k-steps of 4 over the panel width
    const int n64 = (nc + 63) >> 6;
    const int64_t mtiles = (rr + 7) >> 3;
    for (int grp = 0; grp < n64; ++grp) {
      double bf[KS][8];
      int colb[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) colb[j] = grp * 64 + j * 8;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = ks * 4 + t, cn = colb[j] + g;
          bf[ks][j] = (k < NB && cn < nc) ? S.part[k * 256 + cn] : 0.0;
        }
      for (int64_t mt = warp; mt < mtiles; mt += kWarps) {
        const int64_t row = mt * 8 + g;
        const bool rok = row < rr;
        double af[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int k = ks * 4 + t;
          af[ks] = (k < NB && mt * 8 + g < rr) ? S.Ps[(size_t)k * S.rs + mt * 8 + g] : 0.0;
        }
        double c[8][2];
        double* arow = Ab + row * lda + c0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int cb = colb[j] + 2 * t;
          c[j][0] = (rok && cb < nc) ? arow[cb] : 0.0;
          c[j][1] = (rok && cb + 1 < nc) ? arow[cb + 1] : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], af[ks], bf[ks][j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int cb = colb[j] + 2 * t;
          if (rok && cb < nc) arow[cb] = c[j][0];
          if (rok && cb + 1 < nc) arow[cb + 1] = c[j][1];
        }
      }
    }
    __syncthreads();
  }
}

// Blocked Householder QR of block rows [0, r) of A (row-major, ld = ldm,
// even): V below the diagonal, R on and above it; T factors to Tq.
template <int NB>
__device__ void factor_block(const Smem<NB>& S, double* A, int64_t ldm, int64_t r, int l,
                             double* Tq) {
  const int npan = (l + NB - 1) / NB;
  for (int pi = 0; pi < npan; ++pi) {
    const int p0 = pi * NB, nbc = min(NB, l - p0);
    const int64_t rr = r - p0;
    load_panel<NB>(S, A, ldm, p0, r, nbc);
    __syncthreads();
    factor_panel<NB>(S, rr, nbc);
    // panel back to global (V below the diagonal, R on and above it)
    for (int64_t i = threadIdx.x / NB; i < rr; i += kThreads / NB) {
      const int k = threadIdx.x % NB;
      if (k < nbc) A[(p0 + i) * ldm + p0 + k] = S.Ps[(size_t)k * S.rs + i];
    }
    __syncthreads();
    build_T<NB>(S, rr, nbc, true);
    for (int idx = threadIdx.x; idx < NB * NB; idx += kThreads)
      Tq[(size_t)pi * NB * NB + idx] = S.Ts[idx];
    if (p0 + nbc < l) apply_wy<NB, true>(S, A, ldm, p0, r, p0 + nbc, l);
    __syncthreads();
  }
}

// E (r x l, ld lde) <- Q_block E: the block's reflectors, last panel first.
template <int NB>
__device__ void apply_block_q(const Smem<NB>& S, const double* A, int64_t ldm, int64_t r, int l,
                              const double* Tq, double* E, int64_t lde) {
  const int npan = (l + NB - 1) / NB;
  for (int pi = npan - 1; pi >= 0; --pi) {
    const int p0 = pi * NB, nbc = min(NB, l - p0);
    const int64_t rr = r - p0;
    load_panel<NB>(S, A, ldm, p0, r, nbc);
    for (int idx = threadIdx.x; idx < NB * NB; idx += kThreads)
      S.Ts[idx] = Tq[(size_t)pi * NB * NB + idx];
    __syncthreads();
    build_T<NB>(S, rr, nbc, false);
    __syncthreads();
    apply_wy<NB, false>(S, E, lde, p0, r, 0, l);
  }
}

template <int NB>
__global__ void __launch_bounds__(kThreads, 2) tsqr_factor_kernel(Plan P, const double* __restrict__ X,
                                                             int64_t ldx, double* __restrict__ R,
                                                             int64_t ldr, const int* flag) {
  if (flag && *flag == 0) return;
  extern __shared__ __align__(16) double smem_tsqr[];
  const Smem<NB> S = carve<NB>(smem_tsqr, P.rmax);
  cg::grid_group grid = cg::this_grid();
  const int l = P.l;
  const int64_t ldm = P.ldm;
  for (int L = 0; L < P.levels; ++L) {
    const Level& lv = P.lv[L];
    for (int64_t q = blockIdx.x; q < lv.nblk; q += gridDim.x) {
      int64_t s, e;
      block_rows(lv, q, s, e);
      const int64_t r = e - s;
      double* A = lv.M + s * ldm;
      if (L == 0) {  // the leaf's rows of X, one warp per row
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int64_t i = warp; i < r; i += kWarps)
          for (int c = lane; c < l; c += 32) A[i * ldm + c] = X[(s + i) * ldx + c];
        __syncthreads();
      }
      factor_block<NB>(S, A, ldm, r, l, lv.T + (size_t)q * P.npan * NB * NB);
      const bool top = L + 1 == P.levels;
      double* dst = top ? R : P.lv[L + 1].M + q * l * ldm;
      const int64_t ldd = top ? ldr : ldm;
      {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int i = warp; i < l; i += kWarps)
          for (int c = lane; c < l; c += 32) dst[i * ldd + c] = c >= i ? A[(int64_t)i * ldm + c] : 0.0;
      }
      __syncthreads();
    }
    if (L + 1 < P.levels) grid.sync();
  }
}

// Ein: the top block's l x l input (identity when null); Q: rows x lpad.
template <int NB>
__global__ void __launch_bounds__(kThreads, 2) tsqr_q_kernel(Plan P, const double* __restrict__ Ein,
                                                        int64_t lde, double* __restrict__ Q,
                                                        int64_t ldq, int lpad, const int* flag) {
  if (flag && *flag == 0) return;
  extern __shared__ __align__(16) double smem_tsqr[];
  const Smem<NB> S = carve<NB>(smem_tsqr, P.rmax);
  cg::grid_group grid = cg::this_grid();
  const int l = P.l;
  const int64_t ldm = P.ldm;
  for (int L = P.levels - 1; L >= 0; --L) {
    const Level& lv = P.lv[L];
    const bool top = L + 1 == P.levels;
    double* out = L == 0 ? Q : P.Qb[L & 1];
    const int64_t ldo = L == 0 ? ldq : ldm;
    const double* in = top ? Ein : P.Qb[(L + 1) & 1];
    const int64_t ldi = top ? lde : ldm;
    for (int64_t q = blockIdx.x; q < lv.nblk; q += gridDim.x) {
      int64_t s, e;
      block_rows(lv, q, s, e);
      const int64_t r = e - s;
      double* E = out + s * ldo;
      const double* Ei = top ? in : in + q * l * ldi;
      const int wcols = L == 0 ? lpad : l;
      {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int64_t i = warp; i < r; i += kWarps)
          for (int c = lane; c < wcols; c += 32) {
            double v = 0.0;
            if (i < l && c < l) v = Ei ? Ei[i * ldi + c] : (i == c ? 1.0 : 0.0);
            E[i * ldo + c] = v;
          }
      }
      __syncthreads();
      apply_block_q<NB>(S, lv.M + s * ldm, ldm, r, l, lv.T + (size_t)q * P.npan * NB * NB, E, ldo);
      __syncthreads();
    }
    if (L > 0) grid.sync();
  }
}

// dst (drows x dcols) <- src (rows x cols) with zero fill, when *flag != 0
__global__ void pad_copy_kernel(const double* __restrict__ src, int64_t lds, int64_t rows,
                                int cols, double* __restrict__ dst, int64_t ldd, int64_t drows,
                                int dcols, const int* flag) {
  if (flag && *flag == 0) return;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < drows * dcols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / dcols;
    const int c = (int)(idx - i * dcols);
    dst[i * ldd + c] = (i < rows && c < cols) ? src[i * lds + c] : 0.0;
  }
}

void launch_pad_copy(const double* src, int64_t lds, int64_t rows, int cols, double* dst,
                     int64_t ldd, int64_t drows, int dcols, const int* flag, cudaStream_t st) {
  const int64_t n = drows * dcols;
  if (n <= 0) return;
  pad_copy_kernel<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), 1024), 256, 0, st>>>(
      src, lds, rows, cols, dst, ldd, drows, dcols, flag);
  check_launch("tsqr_pad_copy");
}

int pick_nb(int l) {
  for (int nb : {16, 8, 4, 2}) {
    const int rmax = std::max(512, 2 * l);
    size_t need = 0;
    switch (nb) {
      case 16: need = smem_doubles<16>(rmax); break;
      case 8: need = smem_doubles<8>(rmax); break;
      case 4: need = smem_doubles<4>(rmax); break;
      default: need = smem_doubles<2>(rmax); break;
    }
    if (need * 8 <= max_dyn_smem()) return nb;
  }
  return 0;
}

size_t smem_bytes(int nb, int rmax) {
  switch (nb) {
    case 16: return smem_doubles<16>(rmax) * 8;
    case 8: return smem_doubles<8>(rmax) * 8;
    case 4: return smem_doubles<4>(rmax) * 8;
    default: return smem_doubles<2>(rmax) * 8;
  }
}

// The tree's shape for `rows` x l and its workspace layout (doubles).
struct HostPlan {
  Plan p;
  size_t doubles = 0;
};

HostPlan make_plan(int64_t rows, int l, double* work) {
  HostPlan h;
  Plan& p = h.p;
  p.l = l;
  p.nb = pick_nb(l);
  XB_REQUIRE(p.nb > 0, XB_EUNSUPPORTED,
             "TSQR: l = " + std::to_string(l) + " columns exceed the shared-memory panel");
  XB_REQUIRE(rows >= l, XB_ESHAPE, "TSQR needs rows >= cols");
  p.npan = (l + p.nb - 1) / p.nb;
  p.rmax = std::max(512, 2 * l);
  p.ldm = (int)round_up(l, 2);
  p.rows = rows;
  const int64_t G = std::max<int64_t>(2, p.rmax / l);
  size_t off = 0;
  auto take = [&](size_t n) {
    double* q = work ? work + off : nullptr;
    off += (n + 31) / 32 * 32;
    return q;
  };
  int L = 0;
  int64_t units = rows, usize = 1;
  int64_t rows1 = 0;
  while (true) {
    XB_REQUIRE(L < kMaxLevels, XB_EUNSUPPORTED, "TSQR: tree too deep");
    Level& lv = p.lv[L];
    lv.units = units;
    lv.usize = usize;
    lv.nblk = L == 0 ? std::max<int64_t>(1, ceil_div(rows, (int64_t)p.rmax))
                     : ceil_div(units, G);
    lv.M = take((size_t)units * usize * p.ldm);
    lv.T = take((size_t)lv.nblk * p.npan * p.nb * p.nb);
    if (L == 1) rows1 = units * usize;
    ++L;
    if (lv.nblk == 1) break;
    units = lv.nblk;
    usize = l;
  }
  p.levels = L;
  p.Qb[0] = take((size_t)std::max<int64_t>(rows1, 1) * p.ldm);
  p.Qb[1] = take((size_t)std::max<int64_t>(rows1, 1) * p.ldm);
  h.doubles = off;
  return h;
}

template <int NB>
void launch_pass(bool factor, const Plan& p, const double* X, int64_t ldx, double* R, int64_t ldr,
                 const double* Ein, int64_t lde, double* Q, int64_t ldq, int lpad, const int* flag,
                 cudaStream_t st) {
  const size_t sm = smem_bytes(NB, p.rmax);
  const void* fn = factor ? reinterpret_cast<const void*>(&tsqr_factor_kernel<NB>)
                          : reinterpret_cast<const void*>(&tsqr_q_kernel<NB>);
  static bool attr_set[2] = {false, false};
  static size_t attr_bytes[2] = {0, 0};
  if (!attr_set[factor] || attr_bytes[factor] < sm) {
    XB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr_set[factor] = true;
    attr_bytes[factor] = sm;
  }
  int per_sm = 0;
  XB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, sm));
  XB_REQUIRE(per_sm > 0, XB_ECUDA, "TSQR kernel cannot be resident");
  // The Q pass keeps each block's rmax x l slice of Q in L2 between its panel
  // steps (8 read-modify-write passes at l = 120): with two resident CTAs per
  // SM the 296 live blocks (145 MB) spill to DRAM — 12.6 GB of DRAM reads for
  // a 0.96 GB sketch; one per SM: 1e6 x 120 33.4 -> 31.2 ms. (The factor pass
  // is faster with two: 35.9 ms with one.)
  if (!factor) per_sm = 1;
  int64_t most = 1;
  for (int L = 0; L < p.levels; ++L) most = std::max(most, p.lv[L].nblk);
  const int grid = (int)std::min<int64_t>(most, (int64_t)per_sm * kNumSMs);
  Plan pc = p;
  if (factor) {
    void* args[] = {&pc, &X, &ldx, &R, &ldr, &flag};
    XB_CUDA(cudaLaunchCooperativeKernel(fn, grid, kThreads, args, sm, st));
  } else {
    void* args[] = {&pc, &Ein, &lde, &Q, &ldq, &lpad, &flag};
    XB_CUDA(cudaLaunchCooperativeKernel(fn, grid, kThreads, args, sm, st));
  }
  count_launch();
}

void run_pass(bool factor, const Plan& p, const double* X, int64_t ldx, double* R, int64_t ldr,
              const double* Ein, int64_t lde, double* Q, int64_t ldq, int lpad, const int* flag,
              cudaStream_t st) {
  switch (p.nb) {
    case 16: launch_pass<16>(factor, p, X, ldx, R, ldr, Ein, lde, Q, ldq, lpad, flag, st); break;
    case 8: launch_pass<8>(factor, p, X, ldx, R, ldr, Ein, lde, Q, ldq, lpad, flag, st); break;
    case 4: launch_pass<4>(factor, p, X, ldx, R, ldr, Ein, lde, Q, ldq, lpad, flag, st); break;
    default: launch_pass<2>(factor, p, X, ldx, R, ldr, Ein, lde, Q, ldq, lpad, flag, st); break;
  }
}

}  // namespace

size_t tsqr_work_doubles(int64_t rows, int l) { return make_plan(rows, l, nullptr).doubles; }

void launch_tsqr(const double* X, int64_t ldx, int64_t rows, int l, int lpad, double* Q,
                 int64_t ldq, double* R, int64_t ldr, double* work, const int* flag,
                 cudaStream_t st) {
  const HostPlan h = make_plan(rows, l, work);
  run_pass(true, h.p, X, ldx, R, ldr, nullptr, 0, nullptr, 0, 0, flag, st);
  run_pass(false, h.p, nullptr, 0, nullptr, 0, nullptr, 0, Q, ldq, lpad, flag, st);
}

size_t tsqr_sharded_work_doubles(int64_t rows_local, int l, int world) {
  const size_t loc = rows_local >= l ? make_plan(rows_local, l, nullptr).doubles : 0;
  return loc + make_plan((int64_t)world * l, l, nullptr).doubles +
         (size_t)(2 * world + 1) * l * l + 64;
}

// Row-sharded TSQR: local tree -> all-gather of the local R factors -> the
// replicated root over the world*l x l stack -> local Q from this rank's
// slice of the root's Q. `allgather(send, recv, count)` is the
// communicator's stream-ordered all-gather (always called, also when `flag`
// is 0, so every rank issues the same collectives).
void launch_tsqr_sharded(const double* X, int64_t ldx, int64_t rows, int l, int lpad, double* Q,
                         int64_t ldq, double* R, int64_t ldr, double* work, const int* flag,
                         int world, int rank,
                         const std::function<void(const double*, double*, size_t)>& allgather,
                         cudaStream_t st) {
  // fewer local rows than columns: the local "R" is X itself on top of zero
  // rows (the stack's QR is unchanged), and the local Q is the first `rows`
  // rows of this rank's slice of the root's Q
  const bool tree = rows >= l;
  HostPlan loc;
  if (tree) loc = make_plan(rows, l, work);
  double* w2 = work + loc.doubles;
  const HostPlan root = make_plan((int64_t)world * l, l, w2);
  double* Rloc = w2 + root.doubles;
  double* Rall = Rloc + (size_t)l * l;
  double* Qall = Rall + (size_t)world * l * l;
  if (tree)
    run_pass(true, loc.p, X, ldx, Rloc, l, nullptr, 0, nullptr, 0, 0, flag, st);
  else
    launch_pad_copy(X, ldx, rows, l, Rloc, l, l, l, flag, st);
  allgather(Rloc, Rall, (size_t)l * l);
  run_pass(true, root.p, Rall, l, R, ldr, nullptr, 0, nullptr, 0, 0, flag, st);
  run_pass(false, root.p, nullptr, 0, nullptr, 0, nullptr, 0, Qall, l, l, flag, st);
  if (tree)
    run_pass(false, loc.p, nullptr, 0, nullptr, 0, Qall + (size_t)rank * l * l, l, Q, ldq, lpad,
             flag, st);
  else
    launch_pad_copy(Qall + (size_t)rank * l * l, l, rows, l, Q, ldq, rows, lpad, flag, st);
}

}  // namespace xb
