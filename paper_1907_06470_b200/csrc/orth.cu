// Orthonormalisation and small-factor kernels.
//
//  chol_inv      Cholesky G = R^T R of the l x l Gram (f64) and R^{-1}; the
//                core of CholQR2, which replaces the reference's streaming
//                Householder thin_qr (kernels.py:297-351). Both give the
//                unique Q with diag(R) > 0 for a full-rank input.
//  (the Householder fallback for Grams that are not numerically positive
//   definite is the multi-CTA TSQR of tsqr.cu)
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

}  // namespace

size_t max_dyn_smem() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return (size_t)v;
}

namespace {

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

template <typename Tin, typename Tout>
__global__ void copy2d_kernel(const Tin* __restrict__ in, int64_t rows, int64_t cols,
                              int64_t ldin, Tout* __restrict__ out, int64_t ldout) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    out[r * ldout + c] = (Tout)in[r * ldin + c];
  }
}

// x <- (double)(float)x: Omega cast to the float32 storage dtype
// (pipeline.py:281-282) while the sketch buffers stay f64.
__global__ void round_f32_kernel(double* __restrict__ p, int64_t rows, int64_t cols, int64_t ld) {
  const int64_t total = rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / cols, c = idx - r * cols;
    p[r * ld + c] = (double)(float)p[r * ld + c];
  }
}

// M (l x l, ld) := I when *flag (the Householder fallback replaced R^-1 Q).
__global__ void identity_if_kernel(double* __restrict__ M, int64_t ld, int l, const int* flag) {
  if (*flag == 0) return;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)l * l;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / l, c = idx - i * l;
    M[i * ld + c] = (i == c) ? 1.0 : 0.0;
  }
}

__global__ void identity_kernel(double* __restrict__ M, int64_t ld, int l) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)l * l;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / l, c = idx - i * l;
    M[i * ld + c] = (i == c) ? 1.0 : 0.0;
  }
}

// out = ||M||_F (fixed-order block reduction), then M /= out when out > 0
__global__ void __launch_bounds__(1024) frob_normalise_kernel(double* __restrict__ M, int64_t n,
                                                             double* __restrict__ out) {
  __shared__ double part[32];
  __shared__ double nrm;
  double ss = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) ss = fma(M[i], M[i], ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) {
      nrm = sqrt(v);
      *out = nrm;
    }
  }
  __syncthreads();
  if (nrm > 0.0) {
    const double r = 1.0 / nrm;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) M[i] *= r;
  }
}

// gram_path: s_i = sqrt(max(eig_i, 0))^e (pipeline.py:569-571)
__global__ void gram_sigma_kernel(double* __restrict__ s, int l, double e) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < l) {
    const double sp = sqrt(fmax(s[i], 0.0));
    s[i] = e == 1.0 ? sp : pow(sp, e);
  }
}

// V[:, j] /= sqrt(D[j][j]) where D[j][j] > 0 (unit columns, pipeline.py:573-575)
__global__ void scale_cols_kernel(double* __restrict__ V, int64_t ldv, int64_t rows, int k,
                                  const double* __restrict__ D, int64_t ldd) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < rows * k;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / k;
    const int j = (int)(idx - r * k);
    const double d = D[(int64_t)j * ldd + j];
    if (d > 0.0) V[r * ldv + j] /= sqrt(d);
  }
}

}  // namespace

void launch_identity(double* M, int64_t ld, int l, cudaStream_t st) {
  identity_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)l * l, 256), 1024), 256, 0, st>>>(
      M, ld, l);
  check_launch("identity");
}

void launch_frob_normalise(double* M, int64_t n, double* out, cudaStream_t st) {
  frob_normalise_kernel<<<1, 1024, 0, st>>>(M, n, out);
  check_launch("frob_normalise");
}

void launch_gram_sigma(double* s, int l, double exponent, cudaStream_t st) {
  gram_sigma_kernel<<<(l + 255) / 256, 256, 0, st>>>(s, l, exponent);
  check_launch("gram_sigma");
}

void launch_scale_cols_by_diag(double* V, int64_t ldv, int64_t rows, int k, const double* D,
                               int64_t ldd, cudaStream_t st) {
  if (rows <= 0 || k <= 0) return;
  scale_cols_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * k, 256), 4096), 256, 0, st>>>(
      V, ldv, rows, k, D, ldd);
  check_launch("scale_cols");
}

void launch_identity_if(double* M, int64_t ld, int l, const int* flag, cudaStream_t st) {
  identity_if_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)l * l, 256), 1024), 256, 0, st>>>(
      M, ld, l, flag);
  check_launch("identity_if");
}

void launch_deficient(const double* R, int64_t ldr, int l, double eps, int* count, int* cols,
                      cudaStream_t st) {
  deficient_kernel<<<1, kSmallThreads, 0, st>>>(R, ldr, l, eps, count, cols);
  check_launch("deficient");
}

void launch_transpose(const double* in, int64_t rows, int64_t cols, int64_t ldin, double* out,
                      int64_t ldout, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, ldin, out, ldout);
  check_launch("transpose");
}

template <typename Tin, typename Tout>
void launch_copy2d_cast(const Tin* in, int64_t rows, int64_t cols, int64_t ldin, Tout* out,
                        int64_t ldout, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  int blocks = (int)std::min<int64_t>(ceil_div(rows * cols, 256), kNumSMs * 8);
  copy2d_kernel<Tin, Tout><<<blocks, 256, 0, st>>>(in, rows, cols, ldin, out, ldout);
  check_launch("copy2d");
}
template void launch_copy2d_cast<double, double>(const double*, int64_t, int64_t, int64_t, double*,
                                                 int64_t, cudaStream_t);
template void launch_copy2d_cast<float, double>(const float*, int64_t, int64_t, int64_t, double*,
                                                int64_t, cudaStream_t);
template void launch_copy2d_cast<double, float>(const double*, int64_t, int64_t, int64_t, float*,
                                                int64_t, cudaStream_t);

void launch_copy2d(const double* in, int64_t rows, int64_t cols, int64_t ldin, double* out,
                   int64_t ldout, cudaStream_t st) {
  launch_copy2d_cast<double, double>(in, rows, cols, ldin, out, ldout, st);
}

void launch_round_f32(double* p, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  int blocks = (int)std::min<int64_t>(ceil_div(rows * cols, 256), kNumSMs * 8);
  round_f32_kernel<<<blocks, 256, 0, st>>>(p, rows, cols, ld);
  check_launch("round_f32");
}

void launch_zero(double* p, size_t count, cudaStream_t st) {
  XB_CUDA(cudaMemsetAsync(p, 0, count * sizeof(double), st));
}

}  // namespace xb
