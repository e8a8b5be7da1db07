// Sparse A (config 3): CSR SpMM for A*X and A^T*Q, plus the one-time
// device-side format work.
//
// Replaces the reference's sparse products (kernels.py:85-112: per-cell
// bisect + mask + np.add.at; transposed views lexsort every cell,
// pool.py:420-445). Here A arrives once as the reference's SparseBlock COO
// (core.py:245-284: (row, col)-sorted, unique), becomes CSR on the device,
// and A^T gets its own CSR built once (counting sort by column, then each
// column segment ordered by row) so both products are gathers with a fixed
// summation order — deterministic, no fp atomics (SURVEY §7 "do not fuse
// cfg3's sparse pair").
//
// spmm_kernel: one warp per output row; lanes own the sketch columns
// (l <= 32*NC), the row's (col, val) entries are fetched 32 at a time by the
// warp and broadcast by shuffle, and every X row read is a coalesced
// 8*l-byte burst. HBM/L2-bound: algorithmic bytes per launch are
// 12*nnz + 8*(rows+1) + 8*l*(cols_in + rows_out).
#include <algorithm>

#include "common.cuh"

namespace xb {
namespace {

template <int NC>
__global__ void __launch_bounds__(256)
    spmm_kernel(int64_t rows, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ X, int64_t ldx,
                double* __restrict__ Y, int64_t ldy, int l) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < rows; i += nwarps) {
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      int32_t cj = 0;
      double vj = 0.0;
      if (e < e1) {
        cj = __ldg(col + e);
        vj = __ldg(val + e);
      }
      const int cnt = (e1 - base) < 32 ? (int)(e1 - base) : 32;
#pragma unroll 4
      for (int t = 0; t < cnt; ++t) {
        const int64_t j = __shfl_sync(0xffffffffu, cj, t);
        const double v = __shfl_sync(0xffffffffu, vj, t);
        const double* xr = X + j * ldx;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int cc = lane + 32 * c;
          if (cc < l) acc[c] = fma(v, __ldg(xr + cc), acc[c]);
        }
      }
    }
    double* yr = Y + i * ldy;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int cc = lane + 32 * c;
      if (cc < l) yr[cc] = acc[c];
    }
  }
}

// rowptr[r] = first index with rows[idx] >= r (rows sorted ascending).
__global__ void coo_rowptr_kernel(const int64_t* __restrict__ rows, int64_t nnz, int64_t m,
                                  int64_t* __restrict__ rowptr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= m;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (rows[mid] < r)
        lo = mid + 1;
      else
        hi = mid;
    }
    rowptr[r] = lo;
  }
}

__global__ void narrow_cols_kernel(const int64_t* __restrict__ in, int64_t nnz,
                                   int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (int32_t)in[e];
}

// ---- transpose: counting sort by column --------------------------------------

__global__ void col_count_kernel(const int32_t* __restrict__ col, int64_t nnz,
                                 unsigned long long* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[e], 1ull);  // integer counts: order-independent
}

// Single-block exclusive scan of n+1 counters (n up to a few million: one
// pass of blockDim-wide chunks with a running carry).
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(const unsigned long long* __restrict__ in,
                                                              int64_t n, int64_t* __restrict__ out) {
  __shared__ long long warp_tot[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    long long v = (i < n) ? (long long)in[i] : 0;
    // inclusive warp scan
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
      long long w = (lane < (int)(blockDim.x >> 5)) ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const long long before = carry + (warp > 0 ? warp_tot[warp - 1] : 0);
    if (i < n) out[i] = before + x - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = before + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// Scatter entries to their column segment (slot order arbitrary here; fixed
// by the per-segment sort below).
__global__ void col_scatter_kernel(const int64_t* __restrict__ rowptr, int64_t m,
                                   const int32_t* __restrict__ col, const double* __restrict__ val,
                                   const int64_t* __restrict__ tptr,
                                   unsigned long long* __restrict__ fill,
                                   int32_t* __restrict__ trow, double* __restrict__ tval) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < m; i += nwarps) {
    for (int64_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32) {
      const int32_t j = col[e];
      const int64_t slot = tptr[j] + (int64_t)atomicAdd(fill + j, 1ull);
      trow[slot] = (int32_t)i;
      tval[slot] = val[e];
    }
  }
}

// Order each column segment by row (insertion sort; segments are short:
// cfg3 averages 100 entries), making A^T's CSR — and every SpMM^T sum —
// independent of the scatter's atomic order.
__global__ void segment_sort_kernel(const int64_t* __restrict__ tptr, int64_t n,
                                    int32_t* __restrict__ trow, double* __restrict__ tval) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = tptr[j], e = tptr[j + 1];
    for (int64_t x = b + 1; x < e; ++x) {
      const int32_t r = trow[x];
      const double v = tval[x];
      int64_t y = x - 1;
      while (y >= b && trow[y] > r) {
        trow[y + 1] = trow[y];
        tval[y + 1] = tval[y];
        --y;
      }
      trow[y + 1] = r;
      tval[y + 1] = v;
    }
  }
}

int blocks_for(int64_t work, int per_block) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, per_block), kNumSMs * 16));
}

}  // namespace

void launch_spmm(const Csr& a, const double* X, int64_t ldx, double* Y, int64_t ldy, int l,
                 cudaStream_t st) {
  if (a.rows <= 0) return;
  const int warps_per_block = 8;
  const int blocks = blocks_for(a.rows, warps_per_block);
  const int nc = (l + 31) / 32;
#define XB_SPMM(NC)                                                                          \
  spmm_kernel<NC><<<blocks, 256, 0, st>>>(a.rows, a.rowptr, a.col, a.val, X, ldx, Y, ldy, l); \
  break;
  switch (nc) {
    case 1: XB_SPMM(1)
    case 2: XB_SPMM(2)
    case 3: XB_SPMM(3)
    case 4: XB_SPMM(4)
    case 5: case 6: case 7: case 8: XB_SPMM(8)
    default:
      XB_REQUIRE(nc <= 18, XB_EUNSUPPORTED, "spmm: l > 576");
      XB_SPMM(18)
  }
#undef XB_SPMM
  check_launch("spmm");
}

void launch_coo_to_csr(const int64_t* rows, const int64_t* cols, int64_t nnz, int64_t m,
                       int64_t* rowptr, int32_t* col32, cudaStream_t st) {
  coo_rowptr_kernel<<<blocks_for(m + 1, 256), 256, 0, st>>>(rows, nnz, m, rowptr);
  check_launch("coo_rowptr");
  if (nnz > 0) {
    narrow_cols_kernel<<<blocks_for(nnz, 256), 256, 0, st>>>(cols, nnz, col32);
    check_launch("narrow_cols");
  }
}

void launch_csr_transpose(const Csr& a, int64_t* tptr, int32_t* trow, double* tval,
                          unsigned long long* scratch, cudaStream_t st) {
  const int64_t n = a.cols;
  XB_CUDA(cudaMemsetAsync(scratch, 0, (n + 1) * sizeof(unsigned long long), st));
  if (a.nnz > 0) {
    col_count_kernel<<<blocks_for(a.nnz, 256), 256, 0, st>>>(a.col, a.nnz, scratch);
    check_launch("col_count");
  }
  exclusive_scan_kernel<<<1, 1024, 0, st>>>(scratch, n, tptr);
  check_launch("exclusive_scan");
  XB_CUDA(cudaMemsetAsync(scratch, 0, (n + 1) * sizeof(unsigned long long), st));
  if (a.nnz > 0) {
    col_scatter_kernel<<<blocks_for(a.rows, 8), 256, 0, st>>>(a.rowptr, a.rows, a.col, a.val, tptr,
                                                              scratch, trow, tval);
    check_launch("col_scatter");
    segment_sort_kernel<<<blocks_for(n, 128), 128, 0, st>>>(tptr, n, trow, tval);
    check_launch("segment_sort");
  }
}

}  // namespace xb
