// Shared definitions for the xsvd_b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "xsvd_b200.h"

namespace xb {

// Error carrying an xb_status; thrown inside the library, turned into a
// status + thread-local message at the C boundary.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

// A malformed text input (XB_EPARSE) with its 1-based line (mmio.cu).
struct ParseFaultError : Error {
  int64_t line;
  ParseFaultError(int64_t l, const std::string& m);
};

// The C boundary: run f, turn exceptions into a status + thread-local
// message (xb_last_error). set_last_error lives in engine.cu.
void set_last_error(const std::string& msg);
template <typename F>
int guarded_api(F&& f) {
  try {
    f();
    return XB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return XB_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return XB_ECUDA;
  }
}

#define XB_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      throw ::xb::Error(_e == cudaErrorMemoryAllocation ? XB_ENOMEM : XB_ECUDA,         \
                        std::string(#call) + ": " + cudaGetErrorString(_e) + " @ " +    \
                            __FILE__ + ":" + std::to_string(__LINE__));                 \
    }                                                                                   \
  } while (0)

#define XB_REQUIRE(cond, status, msg)                      \
  do {                                                     \
    if (!(cond)) throw ::xb::Error((status), (msg));       \
  } while (0)

// Every kernel launch goes through this counter (xb_launch_count).
extern thread_local int64_t* g_launch_counter;
inline void count_launch() {
  if (g_launch_counter) ++*g_launch_counter;
}
#ifdef XB_TIMELINE
// Experiment build only (-DXB_TIMELINE, XB_TIMELINE=1): an event after every
// launch on the compute stream; LaunchScope prints the gaps at the end of the
// API call (tools: where a step's time goes beyond the kernels themselves).
struct TimelineEntry {
  const char* what;
  cudaEvent_t ev;
};
extern thread_local std::vector<TimelineEntry>* g_timeline;
extern thread_local cudaStream_t g_timeline_stream;
#endif
inline void check_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    throw Error(XB_ECUDA, std::string("launch ") + what + ": " + cudaGetErrorString(e));
#ifdef XB_TIMELINE
  if (g_timeline) {
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, g_timeline_stream);
    g_timeline->push_back({what, ev});
  }
#endif
}

// Experiment knobs (tile shapes, thresholds, timing-only debug modes used by
// tools/): read from the environment ONLY in an experiment build
// (XB_BUILD_EXPERIMENTS=1 python -m paper_1907_06470_b200.build). The release
// library ignores every one of them and runs the defaults, so no stray
// variable can change results or skip work. XB_TRACE (stderr tracing only)
// is read directly.
inline const char* knob(const char* name) {
#ifdef XB_EXPERIMENTS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}
inline bool experiments_build() {
#ifdef XB_EXPERIMENTS
  return true;
#else
  return false;
#endif
}

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
__host__ __device__ inline int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

constexpr int kNumSMs = 148;  // B200

// ---- kernels (host launchers) ----------------------------------------------

// Omega generator: out[r*ld + c] for r < rows, c < cols; columns in
// [cols, ld_pad) are zero-filled when ld_pad > cols.
template <typename T>
void launch_gaussian(uint64_t seed, int64_t row0, int64_t rows, int64_t cols, T* out, int64_t ld,
                     int64_t ld_pad, cudaStream_t st);
void launch_uniform_bits(uint64_t seed, int64_t row0, int64_t rows, int64_t cols, uint64_t* out,
                         cudaStream_t st);

// FP64 DMMA GEMM. C[M x N] = op(A) * B where op(A)=A (A: M x K, lda) or
// A^T (A: K x M, lda); B: K x N (ldb). Split-K over `splits` slices through
// `work` (splits * M * ldc doubles) reduced in slice order (deterministic).
struct DGemmArgs {
  bool trans_a;
  int64_t M, N, K;
  const void* A;  // double, or float when a_f32 (widened to f64 in the kernel)
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  bool a_f32 = false;
  bool accumulate = false;  // C += op(A) B (fixed order: the streamed tiles' sums)
  // triangle structure (f64 DMMA path only):
  //   1 = only output tiles touching the upper triangle are computed (a Gram
  //       read through its upper triangle; strictly-lower tiles are left
  //       undefined), 2 = B is upper triangular (K is clipped per N-tile)
  int tri = 0;
};
// Deterministic slice-order sum of split-K partials into C (+= if accumulate).
void launch_split_reduce(const double* work, int64_t M, int64_t N, int64_t ldw, int64_t stride,
                         int S, double* C, int64_t ldc, bool accumulate, cudaStream_t st);

// tcgen05 3xTF32 GEMM (tgemm.cu) for float32 A; B and C are f64 and B is
// split into tf32 hi/lo planes (bhi, blo: tgemm_b_floats each).
bool tgemm_supported(const DGemmArgs& g);
int tgemm_plan_splits(const DGemmArgs& g);
size_t tgemm_b_floats(const DGemmArgs& g);
void tgemm(const DGemmArgs& g, int splits, double* work, float* bhi, float* blo, cudaStream_t st);

// FP64 products on the int8 tensor cores (ozgemm.cu, Ozaki slices).
bool oz_enabled();
int oz_slices();
// Row / column slice exponents. wide (optional): set to 1 when some row
// (column) has max |x| > 64 x its RMS (the slices would lose accuracy).
// oz_col_exp scratch: 2 cols words when wide != nullptr, else cols.
// Both exponent sets of A (and the range guard when wide != nullptr) in one
// pass; scratch: oz_both_exp_scratch_bytes(rows, cols) bytes.
size_t oz_both_exp_scratch_bytes(int64_t rows, int64_t cols);
void oz_both_exp(const double* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* erow,
                 int32_t* ecol, void* scratch, int* wide, cudaStream_t st);
void oz_both_exp_f32(const float* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* erow,
                     int32_t* ecol, void* scratch, int* wide, cudaStream_t st);
void oz_row_exp(const double* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* e, int* wide,
                cudaStream_t st);
void oz_col_exp(const double* X, int64_t rows, int64_t cols, int64_t ldx, int32_t* e,
                unsigned long long* scratch, int* wide, cudaStream_t st);
// Right-operand slices of X (K x N, ldx, column exponents e): 64-row
// interleaved tiles, zero padded to np (multiple of 64) x kp (of 32).
void oz_slice_right(const double* X, int64_t K, int64_t N, int64_t ldx, const int32_t* e,
                    int8_t* P, int64_t np, int64_t kp, int S, cudaStream_t st);
// Left-operand slices of X (m x n) in one pass: PR = row-scaled slices of X
// (mp x kpn), PC = column-scaled slices of X^T (np x kpm); 128-row
// interleaved tiles (mp, np multiples of 128 with mp >= kpm, np >= kpn;
// kpn, kpm multiples of 32). Either output may be null.
void oz_slice_both(const double* X, int64_t m, int64_t n, int64_t ldx, const int32_t* er,
                   const int32_t* ec, int8_t* PR, int64_t mp, int64_t kpn, int8_t* PC, int64_t np,
                   int64_t kpm, int S, cudaStream_t st);
size_t oz_workspace_doubles(int64_t M, int64_t N, int64_t K);
// float32 A on the int8 pipe (3 digit slices made inside the GEMM): C = op(A) X
// with eL the row (NN) / column (TN) exponents of A, R / eR the 3 right
// slices of X (oz_slice_right_f, np = round_up(N, ozf_tile_n(N))).
int ozf_tile_n(int64_t N);
int ozf_plan_splits(int64_t M, int64_t N, int64_t K);
size_t ozf_workspace_doubles(int64_t M, int64_t N, int64_t K);
void oz_slice_right_f(const double* X, int64_t K, int64_t N, int64_t ldx, const int32_t* e,
                      int8_t* P, int64_t np, int64_t kp, cudaStream_t st);
void ozf_gemm(const float* A, int64_t lda, bool trans_a, const int32_t* eL, const int8_t* R,
              int64_t np, const int32_t* eR, int64_t M, int64_t N, int64_t K, double* C,
              int64_t ldc, bool accumulate, int splits, double* work, cudaStream_t st);
// C (M x N) = L R: L = left slices (rows_p x kp, 128-row interleaved tiles,
// row exponents eL), R = right slices (np x kp, 64-row tiles, column
// exponents eR).
// tri 1: C is a Gram (only tiles on / above the diagonal are computed; the
// rest of C is left unspecified); tri 2: R is upper triangular.
void ozgemm(const int8_t* L, int64_t rows_p, int64_t kp, const int32_t* eL, const int8_t* R,
            int64_t np, const int32_t* eR, int64_t M, int64_t N, int64_t K, double* C, int64_t ldc,
            bool accumulate, int S, double* work, cudaStream_t st, int tri = 0);

// Returns the number of split-K slices that will be used for this shape.
int dgemm_plan_splits(const DGemmArgs& g);
size_t dgemm_workspace_doubles(const DGemmArgs& g, int splits);
void dgemm(const DGemmArgs& g, int splits, double* work, cudaStream_t st);

// Sparse A in CSR (device pointers): rowptr int64[rows+1], col int32[nnz],
// val f64[nnz]; columns sorted within each row.
struct Csr {
  int64_t rows = 0, cols = 0, nnz = 0;
  const int64_t* rowptr = nullptr;
  const int32_t* col = nullptr;
  const double* val = nullptr;
};
// Y (rows x l, ldy) = A X, X (cols x l, ldx). Deterministic gather SpMM.
void launch_spmm(const Csr& a, const double* X, int64_t ldx, double* Y, int64_t ldy, int l,
                 cudaStream_t st);
// The same over per-row entry ranges [lo[i], hi[i]); accumulate: Y += A X.
void launch_spmm_seg(const Csr& a, const int64_t* lo, const int64_t* hi, const double* X,
                     int64_t ldx, double* Y, int64_t ldy, int l, bool accumulate,
                     cudaStream_t st);
// off[b rows + i] = first entry of row i with column >= b bw, b = 0..nb
// (segments sorted by column).
void launch_seg_split(const Csr& a, int nb, int64_t bw, int64_t* off, cudaStream_t st);
// COO (rows sorted, int64 indices) -> CSR rowptr + int32 columns.
void launch_coo_to_csr(const int64_t* rows, const int64_t* cols, int64_t nnz, int64_t m,
                       int64_t* rowptr, int32_t* col32, cudaStream_t st);
// CSR of A^T (cols x rows): tptr[cols+1], trow[nnz], tval[nnz]; each segment
// ordered by row. scratch: cols+1 counters.
void launch_csr_transpose(const Csr& a, int64_t* tptr, int32_t* trow, double* tval,
                          unsigned long long* scratch, cudaStream_t st);

// Cholesky of the leading l x l block of G (ld = ldg): writes upper R and
// R^{-1} (ld = ldr, zero outside l x l), sets *flag = 1 when a pivot falls
// below tau * G_jj (not numerically positive definite). Diag of R is added
// to rdiag (multiplied in when accumulate != 0).
// ws: chol_work_doubles(l) doubles of device scratch (nullptr: stream-ordered
// allocation per call)
size_t chol_work_doubles(int l);
void launch_chol_inv(const double* G, int64_t ldg, int l, double tau, double* R, double* Rinv,
                     int64_t ldr, int* flag, double* ws, cudaStream_t st);
// TSQR (tsqr.cu): tree Householder QR of X (rows x l) -> Q (rows x lpad, zero
// padding columns), R (l x l upper, diag >= 0); both passes return at once
// when *flag == 0 (flag may be null: always run). Q may alias X.
size_t tsqr_work_doubles(int64_t rows, int l);
void launch_tsqr(const double* X, int64_t ldx, int64_t rows, int l, int lpad, double* Q,
                 int64_t ldq, double* R, int64_t ldr, double* work, const int* flag,
                 cudaStream_t st);
// Row-sharded TSQR (local tree, all-gather of the local R factors, replicated
// root, local Q); `allgather(send, recv, count)` enqueues on st.
size_t tsqr_sharded_work_doubles(int64_t rows_local, int l, int world);
void launch_tsqr_sharded(const double* X, int64_t ldx, int64_t rows, int l, int lpad, double* Q,
                         int64_t ldq, double* R, int64_t ldr, double* work, const int* flag,
                         int world, int rank,
                         const std::function<void(const double*, double*, size_t)>& allgather,
                         cudaStream_t st);
// Deficient-column flags from R (l x l, ldr): |R_jj| <= eps * ||R||_F.
// M (l x l, ld) := identity when *flag != 0
void launch_identity_if(double* M, int64_t ld, int l, const int* flag, cudaStream_t st);
void launch_identity(double* M, int64_t ld, int l, cudaStream_t st);
// gram_path helpers: s_i = sqrt(max(s_i, 0))^exponent; V[:, j] /= sqrt(D_jj) (D_jj > 0)
void launch_gram_sigma(double* s, int l, double exponent, cudaStream_t st);
void launch_scale_cols_by_diag(double* V, int64_t ldv, int64_t rows, int k, const double* D,
                               int64_t ldd, cudaStream_t st);
// out (device) = ||M||_F over n contiguous doubles; M /= out when out > 0
void launch_frob_normalise(double* M, int64_t n, double* out, cudaStream_t st);
void launch_deficient(const double* R, int64_t ldr, int l, double eps, int* count, int* cols,
                      cudaStream_t st);

// One-sided Jacobi SVD of M = R^T (R: l x l upper, ldr): produces
//   s[l] (descending), Ub (l x l, ldu: columns = sorted, sign-fixed left
//   singular vectors of M), Wk (l x k, ldw: matching right singular vectors,
//   same signs), status (0 ok, 1 no convergence). tol: rotation threshold on
//   |x_p . x_q| / (|x_p| |x_q|); <= 0 selects the f64 default max(1e-15, l eps).
void launch_jacobi_svd(const double* R, int64_t ldr, int l, int k, double* Ub, int64_t ldu,
                       double* s, double* Wk, int64_t ldw, double* work, int* status,
                       cudaStream_t st, double tol = -1.0);

// The sharded factorisation's communicator (comm.cu): stream-ordered sums
// and all-gathers of f64 device buffers. Backends: NCCL (dlopen'ed; the
// production path over NVLink/NVSwitch) and a host-callback backend (the
// caller's own collectives on host copies, e.g. torch.distributed/gloo —
// used to run the real sharded engine with several processes on one GPU).
struct Comm {
  int world = 1, rank = 0;
  virtual ~Comm() {}
  virtual void allreduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
  // recv (world * count) <- every rank's send (count), rank order
  virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
};
void nccl_unique_id(unsigned char out[128]);
Comm* nccl_comm_create(const unsigned char id[128], int world, int rank);
Comm* host_comm_create(int world, int rank, xb_host_collective_fn fn, void* user);

// Opt-in dynamic shared memory per block on the current device.
size_t max_dyn_smem();
// Global scratch (doubles) launch_jacobi_svd needs in `work` for l.
size_t jacobi_work_doubles(int l);

// FP64 pipe peaks (TFLOP/s) from saturating microbenchmarks (peak.cu).
void measure_fp64_peaks(cudaStream_t st, double* dmma_tflops, double* dfma_tflops);
// tcgen05 dense tensor-pipe peaks: int8 TOP/s (kind::i8), bf16 TFLOP/s (kind::f16).
void measure_tc_peaks(cudaStream_t st, double* i8_tops, double* bf16_tflops, int random_data);

// Small helpers
void launch_transpose(const double* in, int64_t rows, int64_t cols, int64_t ldin, double* out,
                      int64_t ldout, cudaStream_t st);
void launch_copy2d(const double* in, int64_t rows, int64_t cols, int64_t ldin, double* out,
                   int64_t ldout, cudaStream_t st);
template <typename Tin, typename Tout>
void launch_copy2d_cast(const Tin* in, int64_t rows, int64_t cols, int64_t ldin, Tout* out,
                        int64_t ldout, cudaStream_t st);
void launch_round_f32(double* p, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st);
void launch_zero(double* p, size_t count, cudaStream_t st);

}  // namespace xb
