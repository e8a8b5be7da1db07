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
// spmm_kernel: one warp per output row gathering whole l-wide X rows with
// 16-byte loads. The gathered rows are nnz * l * 8 bytes — 19.2 GB per cfg3
// product, 16x A's own bytes — so the kernel is bound by gather traffic from
// L2/HBM; algorithmic (compulsory) bytes per launch:
// 12*nnz + 8*(rows+1) + 8*l*(cols_in + rows_out). Column chunks sized for
// L2 residency were measured slower (re-reading A per chunk, and 64-byte
// row segments of a 960-byte-stride Q do not pack into L2 lines).
#include <algorithm>

#include "common.cuh"

namespace xb {
namespace {

// Y = A X, one warp per output row. Lane t owns columns VEC t + 32 VEC h
// (h < NCH): every nonzero gathers its whole l-wide X row as NCH coalesced
// 8- or 16-byte loads per lane. The row's (col, val) pairs stream in 32 at a
// time (evict-first: A is read once) and are broadcast by shuffle; each sum
// runs in the row's column order (deterministic, no atomics).
template <int NCH, int VEC>
__global__ void __launch_bounds__(256)
    spmm_kernel(int64_t rows, const int64_t* __restrict__ seg_lo,
                const int64_t* __restrict__ seg_hi, const int32_t* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ X, int64_t ldx,
                double* __restrict__ Y, int64_t ldy, int l, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < rows; i += nwarps) {
    double acc[NCH][VEC];
#pragma unroll
    for (int h = 0; h < NCH; ++h)
#pragma unroll
      for (int v = 0; v < VEC; ++v) acc[h][v] = 0.0;
    const int64_t e0 = __ldg(seg_lo + i), e1 = __ldg(seg_hi + i);
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      int32_t cj = 0;
      double vj = 0.0;
      if (e < e1) {
        cj = __ldcs(col + e);
        vj = __ldcs(val + e);
      }
      const int cnt = (e1 - base) < 32 ? (int)(e1 - base) : 32;
      // batches of 4 nonzeros: all 4 * NCH loads are issued before the FMAs
      // (the gather is latency-bound; this keeps them in flight together)
      int t = 0;
      for (; t + 4 <= cnt; t += 4) {
        int64_t j[4];
        double a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          j[u] = __shfl_sync(0xffffffffu, cj, t + u);
          a[u] = __shfl_sync(0xffffffffu, vj, t + u);
        }
        double x[4][NCH][VEC];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double* xr = X + j[u] * ldx + VEC * lane;
#pragma unroll
          for (int h = 0; h < NCH; ++h) {
            if (VEC * lane + 32 * VEC * h < l) {
              if (VEC == 2) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(xr + 64 * h));
                x[u][h][0] = v.x;
                x[u][h][VEC - 1] = v.y;
              } else {
                x[u][h][0] = __ldg(xr + 32 * h);
              }
            } else {
#pragma unroll
              for (int v = 0; v < VEC; ++v) x[u][h][v] = 0.0;
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int h = 0; h < NCH; ++h)
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[h][v] = fma(a[u], x[u][h][v], acc[h][v]);
      }
      for (; t < cnt; ++t) {
        const int64_t j = __shfl_sync(0xffffffffu, cj, t);
        const double a = __shfl_sync(0xffffffffu, vj, t);
        const double* xr = X + j * ldx + VEC * lane;
#pragma unroll
        for (int h = 0; h < NCH; ++h) {
          if (VEC * lane + 32 * VEC * h < l) {
            if (VEC == 2) {
              const double2 x = __ldg(reinterpret_cast<const double2*>(xr + 64 * h));
              acc[h][0] = fma(a, x.x, acc[h][0]);
              acc[h][VEC - 1] = fma(a, x.y, acc[h][VEC - 1]);
            } else {
              acc[h][0] = fma(a, __ldg(xr + 32 * h), acc[h][0]);
            }
          }
        }
      }
    }
    double* yr = Y + i * ldy + VEC * lane;
#pragma unroll
    for (int h = 0; h < NCH; ++h) {
      if (VEC * lane + 32 * VEC * h < l) {
        if (VEC == 2) {
          double2 o = make_double2(acc[h][0], acc[h][VEC - 1]);
          if (accumulate) {
            const double2 p = *reinterpret_cast<const double2*>(yr + 64 * h);
            o.x = p.x + o.x;
            o.y = p.y + o.y;
          }
          if (accumulate)
            *reinterpret_cast<double2*>(yr + 64 * h) = o;
          else
            __stcs(reinterpret_cast<double2*>(yr + 64 * h), o);
        } else if (accumulate) {
          yr[32 * h] += acc[h][0];
        } else {
          __stcs(yr + 32 * h, acc[h][0]);
        }
      }
    }
  }
}

// Row-block split of a CSR whose segments are sorted by column index:
// off[b * rows + i] = first entry of row i with col >= b * bw (b <= nb), so
// block b of row i is [off[b rows + i], off[(b+1) rows + i]).
__global__ void seg_split_kernel(int64_t rows, const int64_t* __restrict__ rowptr,
                                 const int32_t* __restrict__ col, int nb, int64_t bw,
                                 int64_t* __restrict__ off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = rowptr[i], e1 = rowptr[i + 1];
    for (int b = 0; b <= nb; ++b) {
      const int64_t key = (int64_t)b * bw;
      int64_t lo = e0, hi = e1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)col[mid] < key) lo = mid + 1; else hi = mid;
      }
      off[(int64_t)b * rows + i] = lo;
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

// Order each column segment by row, making A^T's CSR — and every SpMM^T
// sum — independent of the scatter's atomic order. One warp per segment:
// segments of up to 32 * SEG_K entries sit in registers (cfg3 averages 100)
// and every entry's final slot is its rank, the number of entries with a
// smaller row (rows are unique within a column); longer segments fall back
// to an in-place insertion sort by one lane.
constexpr int SEG_K = 8;

__global__ void __launch_bounds__(256)
    segment_sort_kernel(const int64_t* __restrict__ tptr, int64_t n, int32_t* __restrict__ trow,
                        double* __restrict__ tval) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < n; j += nwarps) {
    const int64_t b = tptr[j], len = tptr[j + 1] - b;
    if (len <= 1) continue;
    if (len <= 32 * SEG_K) {
      const int kc = (int)((len + 31) >> 5);
      int32_t r[SEG_K];
      double v[SEG_K];
#pragma unroll
      for (int k = 0; k < SEG_K; ++k) {
        const int64_t e = lane + 32 * k;
        r[k] = (k < kc && e < len) ? trow[b + e] : INT32_MAX;
        v[k] = (k < kc && e < len) ? tval[b + e] : 0.0;
      }
      int rank[SEG_K];
#pragma unroll
      for (int k = 0; k < SEG_K; ++k) rank[k] = 0;
      for (int k2 = 0; k2 < kc; ++k2) {
        int32_t mine = 0;
#pragma unroll
        for (int k = 0; k < SEG_K; ++k)
          if (k == k2) mine = r[k];
        for (int s = 0; s < 32; ++s) {
          const int32_t o = __shfl_sync(0xffffffffu, mine, s);
#pragma unroll
          for (int k = 0; k < SEG_K; ++k) rank[k] += (o < r[k]) ? 1 : 0;
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < SEG_K; ++k) {
        if (k < kc && lane + 32 * k < len) {
          trow[b + rank[k]] = r[k];
          tval[b + rank[k]] = v[k];
        }
      }
    } else if (lane == 0) {
      for (int64_t x = b + 1; x < b + len; ++x) {
        const int32_t rr = trow[x];
        const double vv = tval[x];
        int64_t y = x - 1;
        while (y >= b && trow[y] > rr) {
          trow[y + 1] = trow[y];
          tval[y + 1] = tval[y];
          --y;
        }
        trow[y + 1] = rr;
        tval[y + 1] = vv;
      }
    }
    __syncwarp();
  }
}

int blocks_for(int64_t work, int per_block) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(work, per_block), kNumSMs * 16));
}

}  // namespace

void launch_spmm_seg(const Csr& a, const int64_t* lo, const int64_t* hi, const double* X,
                     int64_t ldx, double* Y, int64_t ldy, int l, bool accumulate,
                     cudaStream_t st) {
  if (a.rows <= 0 || l <= 0) return;
  XB_REQUIRE(l <= 576, XB_EUNSUPPORTED, "spmm: l > 576");
  // 16-byte loads when every row of X and Y starts 16-byte aligned and l is even
  const bool vec = (ldx % 2 == 0) && (ldy % 2 == 0) && (l % 2 == 0) &&
                   (reinterpret_cast<uintptr_t>(X) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(Y) % 16 == 0);
  const int blocks = blocks_for(a.rows, 8);
  const int acc = accumulate ? 1 : 0;
#define XB_SPMM(NCH, VEC)                                                                      \
  spmm_kernel<NCH, VEC><<<blocks, 256, 0, st>>>(a.rows, lo, hi, a.col, a.val, X, ldx, Y, ldy, l, \
                                                acc)
  if (vec) {
    switch ((l + 63) / 64) {
      case 1: XB_SPMM(1, 2); break;
      case 2: XB_SPMM(2, 2); break;
      case 3: XB_SPMM(3, 2); break;
      case 4: XB_SPMM(4, 2); break;
      default: XB_SPMM(9, 2); break;
    }
  } else {
    switch ((l + 31) / 32) {
      case 1: XB_SPMM(1, 1); break;
      case 2: XB_SPMM(2, 1); break;
      case 3: XB_SPMM(3, 1); break;
      case 4: XB_SPMM(4, 1); break;
      case 5: case 6: case 7: case 8: XB_SPMM(8, 1); break;
      default: XB_SPMM(18, 1); break;
    }
  }
#undef XB_SPMM
  check_launch("spmm");
}

void launch_spmm(const Csr& a, const double* X, int64_t ldx, double* Y, int64_t ldy, int l,
                 cudaStream_t st) {
  launch_spmm_seg(a, a.rowptr, a.rowptr + 1, X, ldx, Y, ldy, l, false, st);
}

void launch_seg_split(const Csr& a, int nb, int64_t bw, int64_t* off, cudaStream_t st) {
  if (a.rows <= 0) return;
  seg_split_kernel<<<blocks_for(a.rows, 256), 256, 0, st>>>(a.rows, a.rowptr, a.col, nb, bw, off);
  check_launch("seg_split");
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
    segment_sort_kernel<<<blocks_for(n, 8), 256, 0, st>>>(tptr, n, trow, tval);
    check_launch("segment_sort");
  }
}

}  // namespace xb
