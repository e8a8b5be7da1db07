// Orthonormalisation and small-factor kernels.
//
//  chol_inv      Cholesky G = R^T R of the l x l Gram (f64) and R^{-1}; the
//                core of CholQR2, which replaces the reference's streaming
//                Householder thin_qr (kernels.py:297-351). Both give the
//                unique Q with diag(R) > 0 for a full-rank input.
//  householder   single-CTA Householder QR used when the Gram is not
//                numerically positive definite (rank-deficient sketches);
//                follows _house / _householder_qr / _apply_reflectors
//                (kernels.py:247-294) so R keeps a non-negative diagonal.
//  deficient     |R_jj| <= eps * ||R||_F flags (kernels.py:327-331).
//  jacobi_svd    one-sided (Hestenes) Jacobi SVD of M = R_B^T, replacing
//                the Golub-Kahan svd_small (kernels.py:542-562) applied to
//                the projected factor; sorting (stable, descending,
//                kernels.py:535) and the sign rule (kernels.py:556-561) are
//                applied on the device.
// All of these touch l x l or (rows x l) data with l <= a few hundred; they
// are latency-bound single-CTA kernels, kept on the device so the whole
// factorisation runs without host round trips.
#include <cfloat>

#include "common.cuh"

namespace xb {
namespace {

constexpr int kSmallThreads = 1024;
constexpr int kSmallWarps = kSmallThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum over kSmallThreads threads; `red` holds kSmallWarps doubles.
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = (lane < kSmallWarps) ? red[lane] : 0.0;
  r = warp_sum(r);
  return r;
}

size_t max_dyn_smem() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return (size_t)v;
}

// ---------------------------------------------------------------------------
// Cholesky + triangular inverse. W is l x l row-major (stride l) in shared
// memory when it fits, else in global scratch `gw`.
__global__ void __launch_bounds__(kSmallThreads, 1)
    chol_inv_kernel(const double* __restrict__ G, int64_t ldg, int l, double tau,
                    double* __restrict__ R, double* __restrict__ Rinv, int64_t ldr,
                    int* __restrict__ flag, double* gw, int use_smem) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double diag0[1024];
  __shared__ double s_inv;
  double* W = use_smem ? sm : gw;
  const int tid = threadIdx.x;
  const int64_t ll = (int64_t)l * l;
  for (int64_t idx = tid; idx < ll; idx += blockDim.x) {
    const int i = (int)(idx / l), j = (int)(idx - (int64_t)i * l);
    W[idx] = (j >= i) ? G[(int64_t)i * ldg + j] : 0.0;
  }
  for (int j = tid; j < l && j < 1024; j += blockDim.x) diag0[j] = G[(int64_t)j * ldg + j];
  __syncthreads();
  // right-looking Cholesky, upper factor, row j of R finalised at step j
  for (int j = 0; j < l; ++j) {
    if (tid == 0) {
      double d = W[(int64_t)j * l + j];
      const double ref = (j < 1024) ? diag0[j] : d;
      if (!(d > tau * ref) || !(d > 0.0)) {
        *flag = 1;
        d = fmax(fabs(ref), DBL_MIN);  // keep going without NaNs; result discarded
      }
      const double piv = sqrt(d);
      W[(int64_t)j * l + j] = piv;
      s_inv = 1.0 / piv;
    }
    __syncthreads();
    const double inv = s_inv;
    for (int c = j + 1 + tid; c < l; c += blockDim.x) W[(int64_t)j * l + c] *= inv;
    __syncthreads();
    const int rem = l - j - 1;
    const int64_t tri = (int64_t)rem * rem;
    for (int64_t idx = tid; idx < tri; idx += blockDim.x) {
      const int ii = (int)(idx / rem), cc = (int)(idx - (int64_t)ii * rem);
      if (cc < ii) continue;
      const int i = j + 1 + ii, c = j + 1 + cc;
      W[(int64_t)i * l + c] -= W[(int64_t)j * l + i] * W[(int64_t)j * l + c];
    }
    __syncthreads();
  }
  // write R (upper) and zero the lower part / padding handled by caller
  for (int64_t idx = tid; idx < ll; idx += blockDim.x) {
    const int i = (int)(idx / l), j = (int)(idx - (int64_t)i * l);
    R[(int64_t)i * ldr + j] = (j >= i) ? W[idx] : 0.0;
  }
  __syncthreads();
  // In-place inverse, bottom-up rows: X = R^{-1} solves R X = I.
  //   X[i][i] = 1/R[i][i];  X[i][c] = -(1/R[i][i]) sum_{p=i+1..c} R[i][p] X[p][c]
  // Row i of W still holds R[i][:] when processed; rows > i already hold X.
  const int warp = tid >> 5, lane = tid & 31;
  for (int i = l - 1; i >= 0; --i) {
    const double rii = W[(int64_t)i * l + i];
    const double inv = 1.0 / rii;
    // columns c > i: warp per column, lanes over p
    double outv = 0.0;
    int myc = -1;
    for (int c = i + 1 + warp; c < l; c += kSmallWarps) {
      double acc = 0.0;
      for (int p = i + 1 + lane; p <= c; p += 32) acc += W[(int64_t)i * l + p] * W[(int64_t)p * l + c];
      acc = warp_sum(acc);
      // stash the result in a register of lane (c / kSmallWarps) % 32... simpler:
      // write after the barrier via a second pass; keep per-warp results in
      // global R scratch row (Rinv row i), which is not read in this pass.
      if (lane == 0) Rinv[(int64_t)i * ldr + c] = -acc * inv;
    }
    (void)outv;
    (void)myc;
    __syncthreads();
    for (int c = i + 1 + tid; c < l; c += blockDim.x) W[(int64_t)i * l + c] = Rinv[(int64_t)i * ldr + c];
    if (tid == 0) W[(int64_t)i * l + i] = inv;
    __syncthreads();
  }
  for (int64_t idx = tid; idx < ll; idx += blockDim.x) {
    const int i = (int)(idx / l), j = (int)(idx - (int64_t)i * l);
    Rinv[(int64_t)i * ldr + j] = (j >= i) ? W[idx] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Householder QR fallback, single CTA, column-major workspaces.
__global__ void __launch_bounds__(kSmallThreads, 1)
    householder_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int l, int lpad,
                       double* __restrict__ Q, int64_t ldq, double* __restrict__ R, int64_t ldr,
                       double* __restrict__ work, const int* __restrict__ flag) {
  if (*flag == 0) return;
  __shared__ double red[kSmallWarps];
  __shared__ double betas[1024];
  __shared__ double s_v0, s_beta, s_mu;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* Wc = work;                       // rows x l, column-major (reflectors + R)
  double* E = work + (int64_t)rows * l;    // rows x l, column-major (Q build)
  for (int64_t idx = tid; idx < rows * l; idx += blockDim.x) {
    const int64_t i = idx / l;
    const int c = (int)(idx - i * l);
    Wc[(int64_t)c * rows + i] = X[i * ldx + c];
  }
  for (int64_t idx = tid; idx < (int64_t)l * l; idx += blockDim.x) {
    const int i = (int)(idx / l), c = (int)(idx - (int64_t)i * l);
    R[(int64_t)i * ldr + c] = 0.0;
  }
  __syncthreads();
  const int steps = (int)((rows < l) ? rows : l);
  for (int j = 0; j < steps; ++j) {
    double* x = Wc + (int64_t)j * rows;
    double part = 0.0;
    for (int64_t i = j + 1 + tid; i < rows; i += blockDim.x) part += x[i] * x[i];
    const double sigma = block_sum(part, red);
    if (tid == 0) {
      const double x0 = x[j];
      double v0 = 1.0, beta, mu;
      if (sigma == 0.0) {
        beta = (x0 >= 0.0) ? 0.0 : 2.0;
        mu = (x0 >= 0.0) ? x0 : -x0;
      } else {
        mu = sqrt(x0 * x0 + sigma);
        v0 = (x0 <= 0.0) ? (x0 - mu) : (-sigma / (x0 + mu));
        beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
      }
      s_v0 = v0;
      s_beta = beta;
      s_mu = mu;
      betas[j < 1024 ? j : 1023] = beta;
    }
    __syncthreads();
    const double v0 = s_v0, beta = s_beta;
    if (sigma != 0.0) {
      const double iv = 1.0 / v0;
      for (int64_t i = j + 1 + tid; i < rows; i += blockDim.x) x[i] *= iv;
    }
    __syncthreads();
    // trailing columns: warp per column
    for (int c = j + 1 + warp; c < l; c += kSmallWarps) {
      double* y = Wc + (int64_t)c * rows;
      double acc = (lane == 0) ? y[j] : 0.0;
      if (sigma != 0.0)
        for (int64_t i = j + 1 + lane; i < rows; i += 32) acc += x[i] * y[i];
      acc = warp_sum(acc) * beta;
      if (lane == 0) y[j] -= acc;
      if (sigma != 0.0)
        for (int64_t i = j + 1 + lane; i < rows; i += 32) y[i] -= acc * x[i];
    }
    __syncthreads();
    if (tid == 0) R[(int64_t)j * ldr + j] = s_mu;
    for (int c = j + 1 + tid; c < l; c += blockDim.x) R[(int64_t)j * ldr + c] = Wc[(int64_t)c * rows + j];
    __syncthreads();
  }
  // Q = H_0 ... H_{l-1} [I; 0], reflectors applied right to left.
  for (int64_t idx = tid; idx < rows * l; idx += blockDim.x) {
    const int c = (int)(idx / rows);
    const int64_t i = idx - (int64_t)c * rows;
    E[idx] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = steps - 1; j >= 0; --j) {
    const double beta = betas[j < 1024 ? j : 1023];
    if (beta == 0.0) continue;
    const double* v = Wc + (int64_t)j * rows;  // v[j] = 1 implicit, v[i>j] stored
    for (int c = j + warp; c < l; c += kSmallWarps) {
      double* y = E + (int64_t)c * rows;
      double acc = (lane == 0) ? y[j] : 0.0;
      for (int64_t i = j + 1 + lane; i < rows; i += 32) acc += v[i] * y[i];
      acc = warp_sum(acc) * beta;
      if (lane == 0) y[j] -= acc;
      for (int64_t i = j + 1 + lane; i < rows; i += 32) y[i] -= acc * v[i];
    }
    __syncthreads();
  }
  for (int64_t idx = tid; idx < rows * lpad; idx += blockDim.x) {
    const int64_t i = idx / lpad;
    const int c = (int)(idx - i * lpad);
    Q[i * ldq + c] = (c < l) ? E[(int64_t)c * rows + i] : 0.0;
  }
}

__global__ void deficient_kernel(const double* __restrict__ R, int64_t ldr, int l, double eps,
                                 int* __restrict__ count, int* __restrict__ cols) {
  __shared__ double red[kSmallWarps];
  double part = 0.0;
  for (int64_t idx = threadIdx.x; idx < (int64_t)l * l; idx += blockDim.x) {
    const int i = (int)(idx / l), c = (int)(idx - (int64_t)i * l);
    const double v = R[(int64_t)i * ldr + c];
    part += v * v;
  }
  const double norm = sqrt(block_sum(part, red));
  if (threadIdx.x == 0) {
    int n = 0;
    for (int j = 0; j < l; ++j)
      if (fabs(R[(int64_t)j * ldr + j]) <= eps * norm) cols[n++] = j;
    *count = n;
  }
}

// ---------------------------------------------------------------------------
// One-sided Jacobi SVD of M = R^T (l x l). X = M stored column-major in shared
// memory (column j of M = row j of R); J (right vectors) in shared memory when
// both fit, else in global `work`.
__global__ void __launch_bounds__(kSmallThreads, 1)
    jacobi_kernel(const double* __restrict__ Rm, int64_t ldr, int l, int k, double* __restrict__ Ub,
                  int64_t ldu, double* __restrict__ s_out, double* __restrict__ Wk, int64_t ldw,
                  double* __restrict__ work, int* __restrict__ status, int j_in_smem, double tol,
                  int max_sweeps) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_rot;
  __shared__ double s_norm[1024];
  __shared__ int s_perm[1024];
  __shared__ int s_sign[1024];
  double* X = sm;
  double* J = j_in_smem ? sm + (int64_t)l * l : work;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ll = (int64_t)l * l;
  for (int64_t idx = tid; idx < ll; idx += blockDim.x) {
    const int c = (int)(idx / l), r = (int)(idx - (int64_t)c * l);
    X[idx] = Rm[(int64_t)c * ldr + r];  // X[:, c] = R[c, :]
    J[idx] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int L2 = l + (l & 1);
  const int npairs = L2 / 2;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < L2 - 1; ++round) {
      for (int pi = warp; pi < npairs; pi += kSmallWarps) {
        // circle method: position 0 fixed, others rotate
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + round) % (L2 - 1); };
        int p = player(pi), q = player(L2 - 1 - pi);
        if (p >= l || q >= l) continue;
        if (p > q) {
          const int tmp = p;
          p = q;
          q = tmp;
        }
        double* xp = X + (int64_t)p * l;
        double* xq = X + (int64_t)q * l;
        double a = 0.0, b = 0.0, gm = 0.0;
        for (int r = lane; r < l; r += 32) {
          const double u = xp[r], v = xq[r];
          a += u * u;
          b += v * v;
          gm += u * v;
        }
        a = warp_sum(a);
        b = warp_sum(b);
        gm = warp_sum(gm);
        if (fabs(gm) > tol * sqrt(a * b) && gm != 0.0) {
          const double zeta = (b - a) / (2.0 * gm);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t);
          const double s = c * t;
          for (int r = lane; r < l; r += 32) {
            const double u = xp[r], v = xq[r];
            xp[r] = c * u - s * v;
            xq[r] = s * u + c * v;
          }
          double* jp = J + (int64_t)p * l;
          double* jq = J + (int64_t)q * l;
          for (int r = lane; r < l; r += 32) {
            const double u = jp[r], v = jq[r];
            jp[r] = c * u - s * v;
            jq[r] = s * u + c * v;
          }
          if (lane == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    const int rotated = s_rot;
    __syncthreads();
    if (!rotated) break;
  }
  if (tid == 0) *status = (sweep >= max_sweeps) ? 1 : 0;
  // singular values = column norms
  for (int c = warp; c < l; c += kSmallWarps) {
    double a = 0.0;
    for (int r = lane; r < l; r += 32) a += X[(int64_t)c * l + r] * X[(int64_t)c * l + r];
    a = warp_sum(a);
    if (lane == 0) s_norm[c] = sqrt(a);
  }
  __syncthreads();
  // stable descending order: rank = #{i: s_i > s_j} + #{i < j: s_i == s_j}
  for (int j = tid; j < l; j += blockDim.x) {
    const double sj = s_norm[j];
    int rank = 0;
    for (int i = 0; i < l; ++i) {
      const double si = s_norm[i];
      rank += (si > sj) || (si == sj && i < j);
    }
    s_perm[rank] = j;
  }
  __syncthreads();
  // sign rule on U_B columns: largest |entry| positive, earliest row on ties
  for (int i = warp; i < l; i += kSmallWarps) {
    const int c = s_perm[i];
    const double sc = s_norm[c];
    const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
    double best = -1.0;
    int brow = 0;
    for (int r = lane; r < l; r += 32) {
      const double v = fabs(X[(int64_t)c * l + r] * inv);
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
    if (lane == 0) s_sign[i] = (X[(int64_t)c * l + brow] * inv < 0.0) ? -1 : 1;
  }
  __syncthreads();
  for (int i = tid; i < l; i += blockDim.x) s_out[i] = s_norm[s_perm[i]];
  for (int64_t idx = tid; idx < ll; idx += blockDim.x) {
    const int r = (int)(idx / l), i = (int)(idx - (int64_t)r * l);
    const int c = s_perm[i];
    const double sc = s_norm[c];
    const double inv = sc > 0.0 ? 1.0 / sc : 0.0;
    Ub[(int64_t)r * ldu + i] = s_sign[i] * X[(int64_t)c * l + r] * inv;
  }
  for (int64_t idx = tid; idx < (int64_t)l * k; idx += blockDim.x) {
    const int r = (int)(idx / k), i = (int)(idx - (int64_t)r * k);
    const int c = s_perm[i];
    Wk[(int64_t)r * ldw + i] = s_sign[i] * J[(int64_t)c * l + r];
  }
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols,
                                 int64_t ldin, double* __restrict__ out, int64_t ldout) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * ldin + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ldout + r] = tile[threadIdx.x][i];
  }
}

__global__ void copy2d_kernel(const double* __restrict__ in, int64_t rows, int64_t cols,
                              int64_t ldin, double* __restrict__ out, int64_t ldout) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    out[r * ldout + c] = in[r * ldin + c];
  }
}

}  // namespace

void launch_chol_inv(const double* G, int64_t ldg, int l, double tau, double* R, double* Rinv,
                     int64_t ldr, int* flag, cudaStream_t st) {
  const size_t bytes = (size_t)l * l * sizeof(double);
  const int use_smem = bytes <= max_dyn_smem() - 16 * 1024;
  double* gw = nullptr;
  if (!use_smem) {
    // the large-l path borrows the Rinv buffer's tail is not safe; allocate
    XB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&gw), bytes, st));
  }
  const size_t dyn = use_smem ? bytes : 0;
  XB_CUDA(cudaFuncSetAttribute(chol_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)dyn));
  chol_inv_kernel<<<1, kSmallThreads, dyn, st>>>(G, ldg, l, tau, R, Rinv, ldr, flag, gw, use_smem);
  check_launch("chol_inv");
  if (gw) XB_CUDA(cudaFreeAsync(gw, st));
}

void launch_householder_fallback(const double* X, int64_t ldx, int64_t rows, int l, int lpad, double* Q,
                                 int64_t ldq, double* R, int64_t ldr, double* work,
                                 const int* flag, cudaStream_t st) {
  householder_kernel<<<1, kSmallThreads, 0, st>>>(X, ldx, rows, l, lpad, Q, ldq, R, ldr, work, flag);
  check_launch("householder");
}

void launch_deficient(const double* R, int64_t ldr, int l, double eps, int* count, int* cols,
                      cudaStream_t st) {
  deficient_kernel<<<1, kSmallThreads, 0, st>>>(R, ldr, l, eps, count, cols);
  check_launch("deficient");
}

void launch_jacobi_svd(const double* R, int64_t ldr, int l, int k, double* Ub, int64_t ldu,
                       double* s, double* Wk, int64_t ldw, double* work, int* status,
                       cudaStream_t st) {
  XB_REQUIRE(l <= 1024, XB_EUNSUPPORTED, "jacobi_svd: l > 1024");
  const size_t lim = max_dyn_smem() - 24 * 1024;  // static smem arrays
  const size_t one = (size_t)l * l * sizeof(double);
  XB_REQUIRE(one <= lim, XB_EUNSUPPORTED,
             "jacobi_svd: l x l factor exceeds shared memory (multi-CTA Jacobi not built yet)");
  const int j_in_smem = 2 * one <= lim;
  const size_t dyn = j_in_smem ? 2 * one : one;
  XB_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)dyn));
  const double tol = fmax(1e-15, (double)l * DBL_EPSILON);
  jacobi_kernel<<<1, kSmallThreads, dyn, st>>>(R, ldr, l, k, Ub, ldu, s, Wk, ldw, work, status,
                                               j_in_smem, tol, 60);
  check_launch("jacobi_svd");
}

void launch_transpose(const double* in, int64_t rows, int64_t cols, int64_t ldin, double* out,
                      int64_t ldout, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, ldin, out, ldout);
  check_launch("transpose");
}

void launch_copy2d(const double* in, int64_t rows, int64_t cols, int64_t ldin, double* out,
                   int64_t ldout, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  int blocks = (int)std::min<int64_t>(ceil_div(rows * cols, 256), kNumSMs * 8);
  copy2d_kernel<<<blocks, 256, 0, st>>>(in, rows, cols, ldin, out, ldout);
  check_launch("copy2d");
}

void launch_zero(double* p, size_t count, cudaStream_t st) {
  XB_CUDA(cudaMemsetAsync(p, 0, count * sizeof(double), st));
}

}  // namespace xb
