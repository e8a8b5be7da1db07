/*
 * xsvd_b200 — C ABI of the B200-native randomized-SVD hot path.
 *
 * Drop-in boundary for the reference package `xsvd` (arXiv 1907.06470,
 * /root/reference/pkg/src/xsvd). The reference is pure Python with no
 * plugin registry: its hot path is the function
 * `randomized_svd` (pipeline.py:442) built from `gaussian_matrix`
 * (pipeline.py:259), `block_multiply` (kernels.py:145), `thin_qr`
 * (kernels.py:297) and `svd_small` (kernels.py:542). Each entry point below
 * replaces one of those; the Python binding is
 * paper_1907_06470_b200/_lib.py (ctypes), and INTEGRATION.md shows the stub
 * a maintainer would add to xsvd itself.
 *
 * Conventions
 *   - every function returns an int status (XB_OK = 0); the message of the
 *     last failure on the calling thread is xb_last_error();
 *   - plain pointers and sizes only; matrices are row-major with an explicit
 *     leading dimension (elements);
 *   - "host" entry points take caller-owned host buffers and return only
 *     after results are in host memory (synchronous); "_dev" entry points
 *     take device pointers on the context's device and are stream-ordered on
 *     the context's compute stream, synchronised before returning;
 *   - one context = one device = one host thread at a time.
 *
 * Status codes map onto the reference exception taxonomy (errors.py):
 *   XB_ESHAPE -> ShapeError, XB_EVALUE -> ValueError, XB_ENOMEM -> BudgetError,
 *   XB_ECONV -> ConvergenceError, XB_EPARSE -> ParseError (with the 1-based
 *   line, returned separately), XB_ECUDA / XB_ENCCL / XB_EUNSUPPORTED -> XsvdError.
 */
#ifndef XSVD_B200_H
#define XSVD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XB_ABI_VERSION 1
/* xb_build_flags() bits */
#define XB_BUILD_EXPERIMENTS 1 /* experiment build: XB_* tuning/debug knobs are read */

enum xb_status {
  XB_OK = 0,
  XB_ESHAPE = 1,
  XB_EVALUE = 2,
  XB_ENOMEM = 3,
  XB_ECONV = 4,
  XB_ECUDA = 5,
  XB_ENCCL = 6,
  XB_EUNSUPPORTED = 7,
  XB_EPARSE = 8
};

/* Precision.DOUBLE / Precision.SINGLE storage dtypes (core.py:26-46). */
enum xb_dtype { XB_F32 = 1, XB_F64 = 2 };

/* Stage slots of stage_seconds[8], in the order of STAGE_NAMES
 * (pipeline.py:33-51): Text Parsing, Preparation of O, O*A^T,
 * Orthogonalization, A^T*Q_r, SVD0 Preparation, SVD0, Postprocessing. */
#define XB_NUM_STAGES 8

typedef struct xb_ctx xb_ctx;

int xb_abi_version(void);
/* XB_BUILD_* bits of this build (0 = release: no environment knobs read). */
int xb_build_flags(void);
const char* xb_last_error(void);

/* Context: device, compute + copy streams, cached workspaces. */
int xb_create(int device, xb_ctx** out);
int xb_destroy(xb_ctx* ctx);
/* Number of kernels this library launched since the context was created
 * (the bench's gpu_launches evidence). */
int64_t xb_launch_count(const xb_ctx* ctx);
/* The context's compute stream (a cudaStream_t), so callers can record
 * CUDA events on the stream the kernels run on. */
void* xb_compute_stream(xb_ctx* ctx);

/* Per-kernel profiling (measurement only; not on the reference interface).
 * When enabled, the large products on A (the dominant tile-GEMM launches)
 * are bracketed by CUDA events on the compute stream. xb_profile_read fills
 * out[0] = seconds summed over those products, out[1] = their count,
 * out[2] = algorithmic FLOPs (2*m*n*l each), out[3] = A bytes they read
 * (m*n*elem each), and resets the accumulators. */
int xb_profile_enable(xb_ctx* ctx, int on);
int xb_profile_read(xb_ctx* ctx, double* out4);
/* As xb_profile_read, plus out[4] = tensor-pipe operations the products
 * issued (2 x multiply-adds, tile padding included: x3 for the 3xTF32 split,
 * x S(S+1)/2 int8 slice pairs for the Ozaki path; 0 for SpMM) and out[5] =
 * the product kind (0 FP64 DMMA, 1 tcgen05 3xTF32, 2 int8-slice Ozaki FP64,
 * 3 CSR SpMM, 4 int8-slice GEMM of float32 A with the slices made in the
 * kernel; the largest seen, -1 if none). Resets the accumulators. */
int xb_profile_read_ext(xb_ctx* ctx, double* out6);
/* Saturating FP64 microbenchmarks on the context's device: TFLOP/s of the
 * DMMA (mma.sync f64) and DFMA pipes — the f64 roofline denominator. */
int xb_fp64_peaks(xb_ctx* ctx, double* dmma_tflops, double* dfma_tflops);
/* Saturating tcgen05 microbenchmarks (one CTA per SM issuing back-to-back
 * M=128 N=256 MMAs from shared memory): dense int8 TOP/s (kind::i8, the
 * pipe the f64/f32 int8-slice GEMMs run on) and bf16 TFLOP/s (kind::f16) —
 * the measured roofline denominator of the int8-slice GEMMs. */
int xb_tc_peaks(xb_ctx* ctx, double* i8_tops, double* bf16_tflops);
/* The same with the operand tiles filled with uniformly random bytes
 * (random_data != 0) instead of small constants: real digit slices toggle
 * every input bit of the tensor core, its power draw rises and the SM clock
 * it sustains falls (B200: ~1.5 GHz instead of ~1.9 GHz), so this is the
 * tensor rate a kernel working on real data can reach on this device. */
int xb_tc_peaks_data(xb_ctx* ctx, int random_data, double* i8_tops, double* bf16_tflops);

/*
 * Full factorization — replaces randomized_svd (pipeline.py:442-625) with
 * re-orthonormalisation after every product (north star).
 *   A      m x n, leading dim lda, dtype `dtype` (HOST memory; pinned memory
 *          is used in place, pageable memory is staged through a ring of
 *          pinned slots filled by host worker threads)
 *   omega  optional n x (k+p) row-major host buffer of `dtype`; NULL means
 *          generate gaussian_band(seed, 0, n, k+p) on the device (rng.py:65)
 *   U      m x k (ldu >= k) `dtype`;  s  k doubles;  V  n x k (ldv >= k).
 *          U and V must not overlap A or omega: the library may write to
 *          them (first touch of their pages) before the factors are ready
 *   deficient  optional int32[k+p]; *ndeficient receives the count of
 *          columns flagged like thin_qr (kernels.py:327-331)
 *   stage_seconds optional double[XB_NUM_STAGES], device-timed
 */
int xb_rsvd_dense(xb_ctx* ctx, int dtype, int64_t m, int64_t n, const void* A, int64_t lda,
                  const void* omega, uint64_t seed, int k, int p, int q,
                  void* U, int64_t ldu, double* s, void* V, int64_t ldv,
                  int32_t* deficient, int* ndeficient, double* stage_seconds);

/* power = "auto" (RsvdConfig.power's default; pipeline.py:295-372,
 * auto_select_q 396-418). Passing q = XB_POWER_AUTO to xb_rsvd_dense,
 * xb_rsvd_dense_dev, xb_rsvd_dense_sharded_dev, xb_rsvd_coo or
 * xb_rsvd_csr_dev runs up to q_max power passes and stops by the reference's
 * rule on nu_q = ||(A A^T)^q A Omega||_F / sqrt(m l): nu_q < tau nu_0, or
 * consecutive ratios nu_q / nu_{q-1} within 1% (nu_0 = 0 stops at q = 0).
 * The raw products' norms are carried through the re-orthonormalised
 * iteration as small triangular factors. xb_set_power_auto sets q_max / tau
 * for the context (defaults 5, 1e-6); xb_last_power reports the last call's
 * chosen q and its nu sequence (up to cap values, *count = how many). The
 * out-of-core streamer does not support XB_POWER_AUTO (XB_EUNSUPPORTED). */
#define XB_POWER_AUTO (-1)
/* RsvdConfig.gram_path (pipeline.py:526-580) for the next factorisations on
 * this context: B^T of the power matrix (Q^T (A A^T)^q A)^T by 2q more thin
 * products, the l x l Gram B B^T factored by Jacobi, sigma = sqrt(eig)^(1/(2q+1)),
 * V = B^T U_B with unit columns. Not supported by the out-of-core streamer. */
int xb_set_gram_path(xb_ctx* ctx, int on);
int xb_set_power_auto(xb_ctx* ctx, int q_max, double tau);
int xb_last_power(xb_ctx* ctx, int* chosen_q, double* nus, int cap, int* count);

/* Out-of-core factorization (the pinned-host tile streamer): A stays in host
 * memory and streams through HBM in row tiles of `tile_rows` (0 = automatic,
 * ~2 GiB tiles), q + 1 fused passes (Y_i = A_i X and W += A_i^T Y_i from one
 * read of each tile). xb_rsvd_dense switches to this path by itself when A
 * does not fit in device memory; this entry point forces it. Replaces the
 * reference's budgeted residency (BlockPool LRU + spill, pool.py:189-221)
 * for the A-larger-than-memory case (config 4). Omega is generated. */
/* Dense A given as the reference's TILE GRID (a StoredMatrix of several
 * tiles, possibly budgeted or backed by a BlockStore: pool.get /
 * read_cell_dense, pool.py:397-418), never assembled in host memory. The
 * library asks for each tile when it streams its row band:
 *   fetch(user, ti, tj, &ld) -> host pointer to the tile (row-major, ld
 *   elements per row), valid until release(user, ti, tj) (release may be
 *   null); row_cuts[0..ntr], col_cuts[0..ntc] are the grid's cuts.
 * A that fits HBM is ingested band by band (the first product computed as
 * bands land); otherwise (or force_stream != 0) the out-of-core streamer
 * runs q + 1 fused passes over the grid. Outputs as xb_rsvd_dense. */
typedef const void* (*xb_tile_fetch_fn)(void* user, int64_t ti, int64_t tj, int64_t* ld);
typedef void (*xb_tile_release_fn)(void* user, int64_t ti, int64_t tj);
int xb_rsvd_dense_tiles(xb_ctx* ctx, int dtype, int64_t m, int64_t n, const int64_t* row_cuts,
                        int ntr, const int64_t* col_cuts, int ntc, xb_tile_fetch_fn fetch,
                        xb_tile_release_fn release, void* user, int force_stream, uint64_t seed,
                        int k, int p, int q, void* U, int64_t ldu, double* s, void* V,
                        int64_t ldv, int32_t* deficient, int* ndeficient,
                        double* stage_seconds);
int xb_rsvd_dense_streamed(xb_ctx* ctx, int dtype, int64_t m, int64_t n, const void* A,
                           int64_t lda, uint64_t seed, int k, int p, int q, int64_t tile_rows,
                           void* U, int64_t ldu, double* s, void* V, int64_t ldv,
                           int32_t* deficient, int* ndeficient, double* stage_seconds);

/* Same factorization with A, omega, U, V, s already in device memory
 * (the HBM-resident measurement; deficient/ndeficient/stage_seconds stay
 * host pointers). Every *_dev entry orders the library's compute stream
 * after the work already queued on the legacy default stream (where e.g.
 * torch produces the inputs); producers on other streams must be
 * synchronised by the caller. */
int xb_rsvd_dense_dev(xb_ctx* ctx, int dtype, int64_t m, int64_t n, const void* dA, int64_t lda,
                      const void* d_omega, uint64_t seed, int k, int p, int q,
                      void* dU, int64_t ldu, double* d_s, void* dV, int64_t ldv,
                      int32_t* deficient, int* ndeficient, double* stage_seconds);

/*
 * Multi-GPU, row-block sharding (the reference itself has no
 * distributed path). One process per GPU: rank 0 calls xb_comm_unique_id,
 * the 128 bytes are broadcast out of band (e.g. torch.distributed), every
 * rank calls xb_comm_init. Rank g then passes its m_local rows of the
 * m_global x n matrix A; Omega and V are replicated, U is returned for the
 * local rows. A^T Q partials (n x l) and the l x l Grams of the row-sharded
 * sketch are summed with NCCL all-reduce on the compute stream.
 */
int xb_comm_unique_id(unsigned char* out128);
int xb_comm_init(xb_ctx* ctx, const unsigned char* id128, int world, int rank);
/* Host-callback communicator (instead of NCCL): the library copies the
 * operand to host memory and calls fn(user, op, buf, count) with
 *   op XB_COLL_ALLREDUCE_SUM: buf holds count doubles, sum them over ranks
 *                             in place;
 *   op XB_COLL_ALLGATHER:     buf holds world*count doubles, this rank's
 *                             slice at rank*count filled; fill the others.
 * fn returns 0 on success. Used to run the sharded engine with several
 * processes (any transport, e.g. torch.distributed gloo) — one GPU each or
 * several sharing one GPU, since ranks only meet on the host. */
#define XB_COLL_ALLREDUCE_SUM 0
#define XB_COLL_ALLGATHER 1
typedef int (*xb_host_collective_fn)(void* user, int op, double* buf, int64_t count);
int xb_comm_init_host(xb_ctx* ctx, int world, int rank, xb_host_collective_fn fn, void* user);
int xb_rsvd_dense_sharded_dev(xb_ctx* ctx, int dtype, int64_t m_global, int64_t n,
                              int64_t m_local, const void* dA, int64_t lda, uint64_t seed, int k,
                              int p, int q, void* dU, int64_t ldu, double* d_s, void* dV,
                              int64_t ldv, int32_t* deficient, int* ndeficient,
                              double* stage_seconds);

/* Column-block sharding (SURVEY §8e, config 5's layout): rank g passes its
 * columns [col0, col0 + n_local) of the m x n_global matrix A (m x n_local,
 * leading dim lda). Y_g = A_g Omega_g partials (m x l) are summed with one
 * NCCL all-reduce per product over A; Z_g = A_g^T Q is local, and the l x l
 * Grams of the row-sharded n-side sketches (Z, B^T) are summed the same way.
 * Omega_g = rows [col0, col0 + n_local) of gaussian_band(seed, 0, n_global,
 * k + p). U (m x k) and s are replicated; V is returned for the local rows. */
int xb_rsvd_dense_colsharded_dev(xb_ctx* ctx, int dtype, int64_t m, int64_t n_global,
                                 int64_t n_local, int64_t col0, const void* dA, int64_t lda,
                                 uint64_t seed, int k, int p, int q, void* dU, int64_t ldu,
                                 double* d_s, void* dV, int64_t ldv, int32_t* deficient,
                                 int* ndeficient, double* stage_seconds);

/*
 * Sparse A — replaces randomized_svd on a SPARSE StoredMatrix, i.e. the
 * sparse x dense and dense x sparse products of kernels.py:85-112 (Y = A X,
 * Z = A^T Q via a once-built CSR of A^T, B^T = A^T Q). A arrives as the
 * reference's SparseBlock COO (core.py:245-284): int64 rows/cols,
 * (row, col)-sorted without duplicates, float64 values (Precision.DOUBLE).
 * Host buffers; same outputs as xb_rsvd_dense.
 */
/* 1 in *sorted when the COO entries are strictly increasing in (row, col) —
 * the reference's SparseBlock invariant (core.py:245-284) that xb_rsvd_coo and
 * xb_spmm_coo rely on; scanned on host threads. */
int xb_coo_sorted(const int64_t* rows, const int64_t* cols, int64_t nnz, int* sorted);

/* Row-sharded sparse A (config 3's layout): this rank's m_local
 * rows of the m_global x n matrix as device CSR (rowptr int64[m_local + 1]
 * relative to the rank's first row, col int32, val f64). Y = A_g X is local,
 * the n x l partials A_g^T Q_g are summed by the communicator; Omega and V
 * replicated, U for the local rows. */
int xb_rsvd_csr_sharded_dev(xb_ctx* ctx, int64_t m_global, int64_t n, int64_t m_local,
                            int64_t nnz, const int64_t* d_rowptr, const int32_t* d_col,
                            const double* d_val, uint64_t seed, int k, int p, int q, double* dU,
                            int64_t ldu, double* d_s, double* dV, int64_t ldv,
                            int32_t* deficient, int* ndeficient, double* stage_seconds);
int xb_rsvd_coo(xb_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                const int64_t* cols, const double* vals, const double* omega, uint64_t seed,
                int k, int p, int q, double* U, int64_t ldu, double* s, double* V, int64_t ldv,
                int32_t* deficient, int* ndeficient, double* stage_seconds);
/* Device-resident CSR variant: rowptr int64[m+1], col int32[nnz] (sorted
 * within rows), val f64[nnz]; U, s, V device pointers. */
int xb_rsvd_csr_dev(xb_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* d_rowptr,
                    const int32_t* d_col, const double* d_val, const double* d_omega,
                    uint64_t seed, int k, int p, int q, double* dU, int64_t ldu, double* d_s,
                    double* dV, int64_t ldv, int32_t* deficient, int* ndeficient,
                    double* stage_seconds);
/* Matrix Market coordinate input (formats.py:143-323, 381-395), parsed
 * natively with `threads` host threads (0 = all). Triplets are 0-based, in
 * the reference's order (per `chunk_lines` body lines, 0 = 500000: the
 * chunk's entries in file order, then its mirrored off-diagonal entries when
 * the file is symmetric); duplicates are NOT summed here (the pool /
 * device CSR builder does that). Malformed input returns XB_EPARSE with the
 * 1-based line in *err_line and the reference's message in xb_last_error.
 * Feed the arrays to xb_rsvd_coo / xb_spmm_coo (sorted by the library) or
 * register them in a pool; release with xb_coo_free. field: 0 real,
 * 1 integer, 2 pattern (values 1.0). */
typedef struct {
  int64_t rows, cols, nnz;
  int64_t* r;
  int64_t* c;
  double* v;
  int field, symmetric;
} xb_coo;
int xb_mm_info(const char* path, int64_t* rows, int64_t* cols, int64_t* entries, int* field,
               int* symmetric, int64_t* err_line);
int xb_mm_read(const char* path, int threads, int64_t chunk_lines, xb_coo* out,
               int64_t* err_line);
void xb_coo_free(xb_coo* coo);

/* Sparse product step (block_multiply with a sparse left operand,
 * kernels.py:85-97, or its transposed view, pool.py:420-445): Y = op(A) X
 * with op(A) = A (trans = 0, X n x l, Y m x l) or A^T (trans = 1, X m x l,
 * Y n x l). COO as above; host buffers, row-major, f64. */
int xb_spmm_coo(xb_ctx* ctx, int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                const int64_t* cols, const double* vals, int trans, const double* X, int64_t l,
                double* Y);

/* Omega generator — replaces gaussian_band (rng.py:38-70): rows
 * [row0, row0+rows) x cols of N(0,1), cast to `dtype`, row-major `ld`.
 * The uint64 hash stage is bit-exact; log/sin/cos are within a few ulp. */
int xb_gaussian(xb_ctx* ctx, int dtype, uint64_t seed, int64_t row0, int64_t rows, int64_t cols,
                void* out, int64_t ld);
/* The integer stage alone: rows x (2*ceil(cols/2)) uint64 words (rng.py:38-47). */
int xb_uniform_bits(xb_ctx* ctx, uint64_t seed, int64_t row0, int64_t rows, int64_t cols,
                    uint64_t* out);

/* Dense product — replaces block_multiply for dense operands
 * (kernels.py:145-193, 80-84): C = op(A) * B with op(A) = A (trans_a = 0,
 * A is m x kdim) or A^T (trans_a = 1, A is kdim x m, the transposed view of
 * pool.py:390-418). B is kdim x n. Host buffers. */
int xb_gemm(xb_ctx* ctx, int dtype, int trans_a, int64_t m, int64_t n, int64_t kdim,
            const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc);
int xb_gemm_dev(xb_ctx* ctx, int dtype, int trans_a, int64_t m, int64_t n, int64_t kdim,
                const void* dA, int64_t lda, const void* dB, int64_t ldb, void* dC, int64_t ldc);

/* Thin QR — replaces thin_qr (kernels.py:297-351): Y (m x r) = Q R with
 * diag(R) >= 0; CholQR2 with an f64 Gram, falling back to Householder when
 * the Gram is not numerically positive definite. R is r x r f64 row-major. */
int xb_thin_qr(xb_ctx* ctx, int dtype, int64_t m, int64_t r, const void* Y, int64_t ldy,
               void* Q, int64_t ldq, double* R, int32_t* deficient, int* ndeficient);

/* Small SVD — replaces svd_small (kernels.py:542-562): B (r x n, r <= n,
 * f64) = U diag(s) V^T, s non-increasing, each U column's largest-|entry|
 * positive (earliest row on ties). U r x r, s r, V n x r. */
/* TSQR (tsqr.cu) of a device Y (m x r, f64, row-major), always run (the
 * factorisations use it as the CholQR fallback): Q (m x r), R (r x r upper,
 * diag >= 0), deficient columns |R_jj| <= eps ||R||_F (kernels.py:327-331);
 * *seconds = the device time of the two tree passes (may be null). */
int xb_tsqr_dev(xb_ctx* ctx, int64_t m, int64_t r, const double* dY, int64_t ldy, double* dQ,
                int64_t ldq, double* dR, int64_t ldr, int32_t* deficient, int* ndeficient,
                double* seconds);
int xb_svd_small(xb_ctx* ctx, int64_t r, int64_t n, const double* B, int64_t ldb,
                 double* U, double* s, double* V);

#ifdef __cplusplus
}
#endif

#endif /* XSVD_B200_H */
