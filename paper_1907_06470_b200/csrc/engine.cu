// rSVD engine and the C ABI (include/xsvd_b200.h).
//
// The factorisation (xb_rsvd_dense*) replaces the reference driver
// randomized_svd (src/pipeline.py:442-625) with the north star's
// re-orthonormalised power iteration ("xsvd-reorth"):
//
//   Omega   = gaussian_band(seed, 0, n, l)                 Preparation of O
//   Y       = A Omega                    (NN DMMA)          O*A^T
//   Q       = CholQR2(Y)                                    Orthogonalization
//   repeat q times:
//     Z = A^T Q  (TN DMMA);  Qz = CholQR2(Z)                O*A^T / Orth.
//     Y = A Qz   (NN DMMA);  Q  = CholQR2(Y)                O*A^T / Orth.
//   B^T     = A^T Q                      (TN DMMA)          A^T*Q_r
//   B^T     = Q_B R_B                    (CholQR2)          SVD0 Preparation
//   R_B^T   = U_B S W^T                  (Jacobi, sorted, sign rule)   SVD0
//   U       = Q U_B[:, :k],  V = Q_B W[:, :k]   (NN DMMA)   Postprocessing
//
// B^T = A^T Q is the reference's B = Q^T A (pipeline.py:550) transposed — the
// TN orientation the paper's own stage names record.
// Everything after A lands in HBM runs on the device with no host round
// trip; stage times come from CUDA events on the compute stream.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cstdlib>
#include <cfloat>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace xb {
thread_local int64_t* g_launch_counter = nullptr;
#ifdef XB_TIMELINE
thread_local std::vector<TimelineEntry>* g_timeline = nullptr;
thread_local cudaStream_t g_timeline_stream = nullptr;
#endif

// Pageable host -> device copies at the link rate. An xsvd caller hands over
// plain numpy arrays: pinning 8 GiB per call (cudaHostRegister + unregister)
// costs more than twice the DMA itself, and a pageable cudaMemcpy is staged by
// the driver on one thread. Here worker threads copy slices of the caller's
// rows into a ring of pinned slots; each slot's DMA runs while the next slots
// fill, so the copy proceeds at min(host memcpy rate, link rate).
struct HostStager {
  static constexpr int kMaxSlots = 16;
  static constexpr size_t kMaxRow = (size_t)64 << 20;  // widest row staged
  int kSlots;
  size_t kSlot, kPiece;
  struct Task {
    char* dst;
    const char* src;
    size_t dpitch, spitch, width;
    int64_t rows;
  };
  char* ring = nullptr;
  cudaEvent_t ev[kMaxSlots] = {};
  bool used[kMaxSlots] = {};
  int next = 0;
  std::vector<std::thread> workers;
  std::mutex mu;
  std::condition_variable cv_work, cv_done;
  std::vector<Task> tasks;
  size_t head = 0;
  int running = 0;
  bool stop = false;

  HostStager(int nthreads, int slots, size_t slot_bytes, size_t piece_bytes)
      : kSlots(std::max(2, std::min(slots, kMaxSlots))), kSlot(slot_bytes), kPiece(piece_bytes) {
    XB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ring), kSlots * kSlot, cudaHostAllocDefault));
    for (int i = 0; i < kSlots; ++i)
      XB_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    for (int t = 0; t < nthreads; ++t) workers.emplace_back([this] { work(); });
  }
  ~HostStager() {
    {
      std::lock_guard<std::mutex> g(mu);
      stop = true;
    }
    cv_work.notify_all();
    for (auto& t : workers) t.join();
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (ring) cudaFreeHost(ring);
  }
  void work() {
    std::unique_lock<std::mutex> lk(mu);
    for (;;) {
      cv_work.wait(lk, [this] { return stop || head < tasks.size(); });
      if (stop) return;
      const Task t = tasks[head++];
      ++running;
      lk.unlock();
      if (t.dpitch == t.width && t.spitch == t.width) {
        std::memcpy(t.dst, t.src, t.width * (size_t)t.rows);
      } else {
        for (int64_t r = 0; r < t.rows; ++r)
          std::memcpy(t.dst + (size_t)r * t.dpitch, t.src + (size_t)r * t.spitch, t.width);
      }
      lk.lock();
      if (--running == 0 && head == tasks.size()) cv_done.notify_all();
    }
  }
  void run(std::vector<Task>&& ts) {
    std::unique_lock<std::mutex> lk(mu);
    tasks = std::move(ts);
    head = 0;
    cv_work.notify_all();
    cv_done.wait(lk, [this] { return head == tasks.size() && running == 0; });
    tasks.clear();
    head = 0;
  }
  // rows [0, rows) of a pageable host matrix (width bytes per row, spitch
  // apart) -> device rows dpitch apart, enqueued on stream s; the host side
  // of every slot has completed on return, the last DMAs may be in flight
  void copy(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width, int64_t rows,
            cudaStream_t s) {
    XB_REQUIRE(width <= kSlot, XB_EUNSUPPORTED, "host stager: row wider than a staging slot");
    const int64_t per_slot = std::max<int64_t>(1, (int64_t)(kSlot / width));
    for (int64_t r0 = 0; r0 < rows; r0 += per_slot) {
      const int64_t h = std::min(per_slot, rows - r0);
      const int slot = next;
      next = (next + 1) % kSlots;
      if (used[slot]) XB_CUDA(cudaEventSynchronize(ev[slot]));
      char* buf = ring + (size_t)slot * kSlot;
      const char* sp = src + (size_t)r0 * spitch;
      std::vector<Task> ts;
      if (spitch == width) {  // contiguous rows: flat byte pieces
        const size_t total = (size_t)h * width;
        for (size_t o = 0; o < total; o += kPiece)
          ts.push_back({buf + o, sp + o, std::min(kPiece, total - o), std::min(kPiece, total - o),
                        std::min(kPiece, total - o), 1});
      } else {
        const int64_t rp = std::max<int64_t>(1, (int64_t)(kPiece / width));
        for (int64_t r = 0; r < h; r += rp)
          ts.push_back({buf + (size_t)r * width, sp + (size_t)r * spitch, width, spitch, width,
                        std::min(rp, h - r)});
      }
      run(std::move(ts));
      char* dp = dst + (size_t)r0 * dpitch;
      if (dpitch == width)
        XB_CUDA(cudaMemcpyAsync(dp, buf, (size_t)h * width, cudaMemcpyHostToDevice, s));
      else
        XB_CUDA(cudaMemcpy2DAsync(dp, dpitch, buf, width, width, h, cudaMemcpyHostToDevice, s));
      XB_CUDA(cudaEventRecord(ev[slot], s));
      used[slot] = true;
    }
  }
  // The other direction: device rows (spitch apart) -> a pageable host matrix
  // (dpitch apart), complete on return. The DMAs run up to kSlots - 1 slots
  // ahead of the worker threads that copy each landed slot out.
  void copy_out(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width,
                int64_t rows, cudaStream_t s) {
    XB_REQUIRE(width <= kSlot, XB_EUNSUPPORTED, "host stager: row wider than a staging slot");
    const int64_t per_slot = std::max<int64_t>(1, (int64_t)(kSlot / width));
    const int64_t nchunks = (rows + per_slot - 1) / per_slot;
    // slots still owned by earlier host->device copies
    for (int i = 0; i < kSlots; ++i)
      if (used[i]) {
        XB_CUDA(cudaEventSynchronize(ev[i]));
        used[i] = false;
      }
    int64_t issued = 0;
    for (int64_t done = 0; done < nchunks; ++done) {
      while (issued < nchunks && issued < done + kSlots - 1) {
        const int64_t r0 = issued * per_slot, h = std::min(per_slot, rows - r0);
        const int slot = (int)(issued % kSlots);
        XB_CUDA(cudaMemcpy2DAsync(ring + (size_t)slot * kSlot, width, src + (size_t)r0 * spitch,
                                  spitch, width, h, cudaMemcpyDeviceToHost, s));
        XB_CUDA(cudaEventRecord(ev[slot], s));
        ++issued;
      }
      const int64_t r0 = done * per_slot, h = std::min(per_slot, rows - r0);
      const int slot = (int)(done % kSlots);
      XB_CUDA(cudaEventSynchronize(ev[slot]));
      const char* buf = ring + (size_t)slot * kSlot;
      char* dp = dst + (size_t)r0 * dpitch;
      std::vector<Task> ts;
      if (dpitch == width) {
        const size_t total = (size_t)h * width;
        for (size_t o = 0; o < total; o += kPiece)
          ts.push_back({dp + o, buf + o, std::min(kPiece, total - o), std::min(kPiece, total - o),
                        std::min(kPiece, total - o), 1});
      } else {
        const int64_t rp = std::max<int64_t>(1, (int64_t)(kPiece / width));
        for (int64_t r = 0; r < h; r += rp)
          ts.push_back({dp + (size_t)r * dpitch, buf + (size_t)r * width, dpitch, width, width,
                        std::min(rp, h - r)});
      }
      run(std::move(ts));
    }
    next = 0;
  }
};
}  // namespace xb

using namespace xb;

struct xb_ctx {
  int device = 0;
  cudaStream_t st = nullptr;  // compute
  cudaStream_t cp = nullptr;  // host <-> device copies
  int64_t launches = 0;
  cudaEvent_t caller_ev = nullptr;  // orders the compute stream after the caller's
  struct Buf {
    void* p;
    size_t bytes;
    uint64_t gen;  // the ABI call that last used it
  };
  std::map<std::string, Buf> bufs;
  uint64_t gen = 0;  // bumped on entry to every ABI call
  std::vector<cudaEvent_t> events;
  // power = "auto" (xb_set_power_auto / xb_last_power): the reference's
  // stopping rule parameters and the last call's outcome
  int auto_qmax = 5;
  double auto_tau = 1e-6;
  int last_q = -1;
  std::vector<double> last_nus;
  // RsvdConfig.gram_path (xb_set_gram_path): project the power matrix and
  // factor its Gram (pipeline.py:526-580)
  bool gram_path = false;
  // per-kernel profiling of the products on A (xb_profile_*)
  bool profiling = false;
  // kind: 0 FP64 DMMA tile GEMM, 1 tcgen05 3xTF32 GEMM, 2 int8-slice
  // (Ozaki) GEMM, 3 CSR SpMM, 4 int8-slice GEMM of float32 A; pipe_ops = tensor-pipe operations issued
  // (multiply-adds x 2, padding included) for the tensor kinds, else 0
  struct ProfMark {
    cudaEvent_t b, e;
    double flops, bytes, pipe_ops;
    int kind;
  };
  std::vector<ProfMark> prof_pending;
  std::vector<cudaEvent_t> prof_pool;
  double prof_acc[6] = {0, 0, 0, 0, 0, -1};

  cudaEvent_t prof_event() {
    if (!prof_pool.empty()) {
      cudaEvent_t e = prof_pool.back();
      prof_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    XB_CUDA(cudaEventCreate(&e));
    return e;
  }
  // resolve recorded marks (call after the stream is synchronised)
  void prof_collect() {
    for (auto& m : prof_pending) {
      float ms = 0.f;
      XB_CUDA(cudaEventElapsedTime(&ms, m.b, m.e));
      prof_acc[0] += ms * 1e-3;
      prof_acc[1] += 1;
      prof_acc[2] += m.flops;
      prof_acc[3] += m.bytes;
      prof_acc[4] += m.pipe_ops;
      prof_acc[5] = std::max(prof_acc[5], (double)m.kind);
      prof_pool.push_back(m.b);
      prof_pool.push_back(m.e);
    }
    prof_pending.clear();
  }

  // Named device buffers cached across calls. When HBM runs out, buffers no
  // earlier step of the current call has touched are released and the
  // allocation retried (a previous call's shapes must not pin memory).
  void* buf(const std::string& name, size_t bytes) {
    auto it = bufs.find(name);
    if (it != bufs.end() && it->second.bytes >= bytes) {
      it->second.gen = gen;
      return it->second.p;
    }
    if (it != bufs.end()) {
      XB_CUDA(cudaStreamSynchronize(st));
      XB_CUDA(cudaFree(it->second.p));
      bufs.erase(it);
    }
    void* p = nullptr;
    const size_t sz = std::max<size_t>(bytes, 256);
    if (cudaMalloc(&p, sz) != cudaSuccess) {
      cudaGetLastError();
      XB_CUDA(cudaStreamSynchronize(st));
      XB_CUDA(cudaStreamSynchronize(cp));
      for (auto i = bufs.begin(); i != bufs.end();) {
        if (i->second.gen != gen) {
          XB_CUDA(cudaFree(i->second.p));
          i = bufs.erase(i);
        } else {
          ++i;
        }
      }
      XB_REQUIRE(cudaMalloc(&p, sz) == cudaSuccess, XB_ENOMEM,
                 "device allocation of " + std::to_string(sz) + " bytes (" + name + ") failed");
    }
    bufs[name] = {p, bytes, gen};
    if (getenv("XB_TRACE")) fprintf(stderr, "[xb] alloc %s %zu B\n", name.c_str(), sz);
    return p;
  }
  size_t buf_bytes(const std::string& name) const {
    auto it = bufs.find(name);
    return it == bufs.end() ? 0 : it->second.bytes;
  }
  size_t cached_bytes() const {
    size_t t = 0;
    for (auto& kv : bufs) t += kv.second.bytes;
    return t;
  }
  double* dbuf(const std::string& name, size_t count) {
    return static_cast<double*>(buf(name, count * sizeof(double)));
  }
  // communicator for the sharded factorisations (xb_comm_init: NCCL;
  // xb_comm_init_host: the caller's host collectives), its stream (the
  // exchanges overlap the products' later row chunks) and events
  Comm* comm = nullptr;
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> xev;
  int world = 1, rank = 0;
  // pageable-host -> device staging (worker threads + pinned ring), created
  // on first use
  xb::HostStager* stager = nullptr;
  int* ibuf(const std::string& name, size_t count) {
    return static_cast<int*>(buf(name, count * sizeof(int)));
  }
};

namespace {

thread_local std::string g_last_error;
// xb_rsvd_dense_streamed sets this for the duration of its call: >= 0 forces
// the out-of-core streamer (0 = automatic tile height)
thread_local int64_t g_force_stream_rows = -1;

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

size_t stage_slot_bytes();
int stage_slots();
size_t stage_piece_bytes();
int stage_threads();

// Device rows -> host rows, stream-ordered after the producers on c->st and
// complete on return. Pinned or small destinations get one DMA; large
// pageable ones go through the staging ring (HostStager::copy_out: the DMAs
// run ahead of the worker threads that copy each landed slot out; a pageable
// cudaMemcpy runs at a fraction of the link rate).
void d2h_rows(xb_ctx* c, void* dst, size_t ld_dst, const void* src, size_t ld_src,
              size_t row_bytes, int64_t rows) {
  const size_t total = row_bytes * (size_t)rows;
  if (rows <= 0 || row_bytes == 0) return;
  if (total < ((size_t)4 << 20) || is_pinned(dst)) {
    XB_CUDA(cudaMemcpy2DAsync(dst, ld_dst, src, ld_src, row_bytes, rows, cudaMemcpyDeviceToHost,
                              c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
    return;
  }
  // large pageable destination: pinned ring + worker threads (HostStager)
  if (row_bytes <= HostStager::kMaxRow) {
    const size_t slot_bytes =
        std::max<size_t>(stage_slot_bytes(), (size_t)round_up((int64_t)row_bytes, 4096));
    if (c->stager && c->stager->kSlot < slot_bytes) {
      delete c->stager;
      c->stager = nullptr;
    }
    if (!c->stager)
      c->stager = new HostStager(stage_threads(), stage_slots(), slot_bytes, stage_piece_bytes());
    c->stager->copy_out(static_cast<char*>(dst), ld_dst, static_cast<const char*>(src), ld_src,
                        row_bytes, rows, c->st);
    return;
  }
  XB_CUDA(cudaMemcpy2DAsync(dst, ld_dst, src, ld_src, row_bytes, rows, cudaMemcpyDeviceToHost,
                            c->st));
  XB_CUDA(cudaStreamSynchronize(c->st));
}

// *_dev entry points take the caller's device buffers: their producers may
// still be running on the caller's legacy default stream (e.g. torch's),
// while the library computes on its own non-blocking stream. Order the
// compute stream after everything already queued there.
void after_caller_stream(xb_ctx* c) {
  if (!c->caller_ev) XB_CUDA(cudaEventCreateWithFlags(&c->caller_ev, cudaEventDisableTiming));
  XB_CUDA(cudaEventRecord(c->caller_ev, cudaStreamLegacy));
  XB_CUDA(cudaStreamWaitEvent(c->st, c->caller_ev, 0));
}

struct LaunchScope {
  int64_t* prev;
  explicit LaunchScope(xb_ctx* c) : prev(g_launch_counter) {
    g_launch_counter = &c->launches;
    ++c->gen;
    cudaSetDevice(c->device);
#ifdef XB_TIMELINE
    if (getenv("XB_TIMELINE") && !g_timeline) {
      g_timeline = new std::vector<TimelineEntry>();
      g_timeline_stream = c->st;
      cudaEvent_t ev;
      cudaEventCreate(&ev);
      cudaEventRecord(ev, c->st);
      g_timeline->push_back({"(start)", ev});
      own_timeline = true;
    }
#endif
  }
  ~LaunchScope() {
    g_launch_counter = prev;
#ifdef XB_TIMELINE
    if (own_timeline) {
      cudaStreamSynchronize(g_timeline_stream);
      auto& v = *g_timeline;
      float total = 0.f;
      if (v.size() > 1) cudaEventElapsedTime(&total, v.front().ev, v.back().ev);
      fprintf(stderr, "[xb timeline] %zu launches, %.3f ms first to last event\n", v.size() - 1,
              total);
      for (size_t i = 1; i < v.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, v[i - 1].ev, v[i].ev);
        fprintf(stderr, "[xb timeline] %3zu %-22s %9.1f us\n", i, v[i].what, ms * 1e3f);
      }
      for (auto& e : v) cudaEventDestroy(e.ev);
      delete g_timeline;
      g_timeline = nullptr;
    }
#endif
  }
#ifdef XB_TIMELINE
  bool own_timeline = false;
#endif
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return XB_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return XB_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return XB_ECUDA;
  }
}

// ---- stage clock -------------------------------------------------------------

enum Stage {
  kParse = 0,
  kGaussian = 1,
  kSketch = 2,
  kOrtho = 3,
  kProject = 4,
  kSvdPrep = 5,
  kSvd = 6,
  kPost = 7
};

struct StageClock {
  xb_ctx* c;
  std::vector<std::pair<int, cudaEvent_t>> marks;
  size_t next_event = 0;
  explicit StageClock(xb_ctx* ctx) : c(ctx) {}
  cudaEvent_t ev() {
    if (next_event >= c->events.size()) {
      cudaEvent_t e;
      XB_CUDA(cudaEventCreate(&e));
      c->events.push_back(e);
    }
    return c->events[next_event++];
  }
  void enter(int stage) {
    if (!marks.empty() && marks.back().first == stage) return;
    cudaEvent_t e = ev();
    XB_CUDA(cudaEventRecord(e, c->st));
    marks.push_back({stage, e});
  }
  // Call after the stream is synchronised.
  void finish(double* out) {
    cudaEvent_t e = ev();
    XB_CUDA(cudaEventRecord(e, c->st));
    XB_CUDA(cudaEventSynchronize(e));
    if (!out) return;
    for (size_t i = 0; i < marks.size(); ++i) {
      cudaEvent_t end = (i + 1 < marks.size()) ? marks[i + 1].second : e;
      float ms = 0.f;
      XB_CUDA(cudaEventElapsedTime(&ms, marks[i].second, end));
      out[marks[i].first] += ms * 1e-3;
    }
  }
};

// ---- building blocks ---------------------------------------------------------

void gemm(xb_ctx* c, bool ta, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
          const double* B, int64_t ldb, double* C, int64_t ldc, int tri = 0) {
  DGemmArgs g{ta, M, N, K, A, lda, B, ldb, C, ldc};
  g.tri = tri;
  const int splits = dgemm_plan_splits(g);
  double* work = nullptr;
  const size_t need = dgemm_workspace_doubles(g, splits);
  if (need) work = c->dbuf("split", need);
  dgemm(g, splits, work, c->st);
}

// Jacobi rotation threshold for the small SVD of a float32 factorisation:
// columns orthogonal to 1e-8 (relative) are far past the f32 targets and
// save the last quadratic sweep (cfg5-like probe, l = 550: 11 -> 10 sweeps,
// sigma 3.86e-8 and angles 2.5e-5 unchanged to 3 digits; cfg5 SVD0 stage
// 38.6 -> 32.2 ms). float64 uses max(1e-15, l eps). (Experiment builds:
// XB_JACOBI_TOL_F32 / XB_JACOBI_TOL_F64 override.)
static double jacobi_tol(bool f32) {
  static const double t = [] {
    const char* e = knob("XB_JACOBI_TOL_F32");
    return e ? atof(e) : 1e-8;
  }();
  static const double t64 = [] {
    const char* e = knob("XB_JACOBI_TOL_F64");
    return e ? atof(e) : -1.0;
  }();
  return f32 ? t : t64;
}

// Slice count of the float32 configs' f64 products on the int8 pipe (n-side
// QR Grams, X R^-1, the V lift). 4 slices carry >= 28 bits, beyond the f32
// data; measured at a cfg5-like 2048 x 65536 (tools/probe_qr_slices.py,
// profiles/r01_qr_slices.md): sigma 3.9e-8 / angle 2.5e-5 at 4 slices vs
// 3.6e-8 / 3.4e-5 at 6 (targets 1e-4 / 1e-3); 3 slices 1.2e-7 / 9.7e-5.
// (Experiment builds: XB_OZ_QR_SLICES overrides.)
static int oz_qr_slices() {
  static const int s = [] {
    const char* e = knob("XB_OZ_QR_SLICES");
    return e ? std::max(3, std::min(6, atoi(e))) : 4;
  }();
  return s;
}

// C = op(A) B for f64 device operands on the int8 tensor pipe (Ozaki
// slices of both operands, ozgemm.cu): exponents, slicing and the GEMM.
// Used for the n-side orthonormalisation products of float32 configs at
// oz_qr_slices() (the 1e-4 / 1e-3 targets leave a large margin) and by the
// XB_GEMM_OZ diagnostics at the f64 count, oz_slices().
void oz_gemm64(xb_ctx* c, bool ta, int64_t m, int64_t n, int64_t kdim, const double* A,
               int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int tri, int S) {
  const int64_t kp = round_up(kdim, 32), np = round_up(n, 64), mp = round_up(m, 128);
  int8_t* L = static_cast<int8_t*>(c->buf("ozg_L", (size_t)S * mp * kp));
  int8_t* R = static_cast<int8_t*>(c->buf("ozg_R", (size_t)S * np * kp));
  int32_t* eL = c->ibuf("ozg_eL", m);
  int32_t* eR = c->ibuf("ozg_eR", np);
  auto* scr = static_cast<unsigned long long*>(c->buf("ozg_scr", (size_t)std::max(m, np) * 8));
  if (ta) {  // op(A) = A^T, A stored kdim x m: column slices of the stored A
    oz_col_exp(A, kdim, m, lda, eL, scr, nullptr, c->st);
    oz_slice_both(A, kdim, m, lda, nullptr, eL, nullptr, round_up(kdim, 128), round_up(m, 32), L,
                  mp, kp, S, c->st);
  } else {
    oz_row_exp(A, m, kdim, lda, eL, nullptr, c->st);
    oz_slice_both(A, m, kdim, lda, eL, nullptr, L, mp, kp, nullptr, round_up(kdim, 128),
                  round_up(m, 32), S, c->st);
  }
  if (ta && A == B && lda == ldb && m == n)  // Gram: the same column exponents
    XB_CUDA(cudaMemcpyAsync(eR, eL, (size_t)m * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->st));
  else
    oz_col_exp(B, kdim, n, ldb, eR, scr, nullptr, c->st);
  oz_slice_right(B, kdim, n, ldb, eR, R, np, kp, S, c->st);
  const size_t wd = oz_workspace_doubles(m, n, kdim);
  double* work = wd ? c->dbuf("split", wd) : nullptr;
  ozgemm(L, mp, kp, eL, R, np, eR, m, n, kdim, C, ldc, false, S, work, c->st, tri);
}

// gemm() or, when `oz` and the big operand has >= 2^24 elements, oz_gemm64
void gemm_big(xb_ctx* c, bool oz, bool ta, int64_t M, int64_t N, int64_t K, const double* A,
              int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int tri = 0) {
  if (oz && oz_enabled() && (double)M * (double)K >= (double)(1 << 24) && M >= 64 && K >= 64)
    oz_gemm64(c, ta, M, N, K, A, lda, B, ldb, C, ldc, tri, oz_qr_slices());
  else
    gemm(c, ta, M, N, K, A, lda, B, ldb, C, ldc, tri);
}

// The caller's A in device memory: f64, or f32 (Precision.SINGLE storage).
struct AView {
  const void* p;
  int64_t ld;
  bool f32;
  size_t esz() const { return f32 ? 4 : 8; }
  const void* rows_from(int64_t r0) const {
    return static_cast<const char*>(p) + (size_t)r0 * ld * esz();
  }
};

// One product: float32 A goes to the tcgen05 3xTF32 kernel (tgemm.cu) when
// its layout allows TMA, everything else to the FP64 DMMA kernel.
void run_gemm(xb_ctx* c, const DGemmArgs& g) {
  if (tgemm_supported(g)) {
    const int splits = tgemm_plan_splits(g);
    double* work = nullptr;
    const size_t need = dgemm_workspace_doubles(g, splits);
    if (need) work = c->dbuf("split", need);
    const size_t nb = tgemm_b_floats(g);
    float* bhi = static_cast<float*>(c->buf("tg_bhi", nb * 4));
    float* blo = static_cast<float*>(c->buf("tg_blo", nb * 4));
    tgemm(g, splits, work, bhi, blo, c->st);
    return;
  }
  const int splits = dgemm_plan_splits(g);
  double* work = nullptr;
  const size_t need = dgemm_workspace_doubles(g, splits);
  if (need) work = c->dbuf("split", need);
  dgemm(g, splits, work, c->st);
}

// A product on A (the dominant kernel): bracketed by events when profiling.
void gemm_on_a(xb_ctx* c, bool ta, int64_t M, int64_t N, int64_t K, const AView& a,
               int64_t row0, const double* B, int64_t ldb, double* C, int64_t ldc, int l) {
  cudaEvent_t b = nullptr, e = nullptr;
  if (c->profiling) {
    b = c->prof_event();
    e = c->prof_event();
    XB_CUDA(cudaEventRecord(b, c->st));
  }
  DGemmArgs g{ta, M, N, K, a.rows_from(row0), a.ld, B, ldb, C, ldc, a.f32};
  run_gemm(c, g);
  if (c->profiling) {
    XB_CUDA(cudaEventRecord(e, c->st));
    const double mn = (double)M * (double)K;  // A is M x K (NN) or K x M (TN)
    const bool tg = tgemm_supported(g);
    c->prof_pending.push_back(
        {b, e, 2.0 * mn * l, mn * a.esz(), (tg ? 3.0 : 1.0) * 2.0 * mn * N, tg ? 1 : 0});
  }
}

struct Small {
  int l, lp;
  double *G, *R1, *R1i, *R2, *R2i, *Rs, *cw;
  int* flag;
  // sharded sketch (rows over ranks): the communicator that sums its Grams
  // and gathers the TSQR fallback's R factors
  Comm* comm = nullptr;
  // float32 configs: the big Gram / X R^-1 products of the single-pass QRs
  // on the int8 pipe (gemm_big)
  bool oz = false;
};

Small small_bufs(xb_ctx* c, int l) {
  Small s;
  s.l = l;
  s.lp = (int)round_up(l, 8);
  const size_t ll = (size_t)s.lp * s.lp;
  s.G = c->dbuf("G", ll);
  s.R1 = c->dbuf("R1", ll);
  s.R1i = c->dbuf("R1i", ll);
  s.R2 = c->dbuf("R2", ll);
  s.R2i = c->dbuf("R2i", ll);
  s.Rs = c->dbuf("Rscratch", ll);
  s.flag = c->ibuf("flag", 4);
  s.cw = c->dbuf("chol_ws", chol_work_doubles(l));
  XB_CUDA(cudaMemsetAsync(s.R1, 0, ll * sizeof(double), c->st));
  XB_CUDA(cudaMemsetAsync(s.R1i, 0, ll * sizeof(double), c->st));
  XB_CUDA(cudaMemsetAsync(s.R2, 0, ll * sizeof(double), c->st));
  XB_CUDA(cudaMemsetAsync(s.R2i, 0, ll * sizeof(double), c->st));
  return s;
}

// Q (rows x lp) = CholQR2(X), zero padding columns l..lp-1 preserved.
// If Rout != null it receives R = R2 R1 (lp x lp, zero padded).
// G = X^T X over this rank's rows, summed over ranks when X is row-sharded.
void gram(xb_ctx* c, const Small& s, const double* X, int64_t rows, bool sharded,
          bool oz = false) {
  // upper-triangle tiles only: the Cholesky kernels read G's upper triangle
  gemm_big(c, oz, true, s.lp, s.lp, rows, X, s.lp, X, s.lp, s.G, s.lp, /*tri=*/1);
  if (sharded) s.comm->allreduce_sum(s.G, (size_t)s.lp * s.lp, c->st);
}

// The fallback when a Cholesky pivot flagged (device-side test, no host
// round trip): TSQR of X recomputes Q and R (tsqr.cu); for a sharded sketch
// the local trees meet through an all-gather of their R factors.
void qr_fallback(xb_ctx* c, const Small& s, const double* X, int64_t rows, double* Q, double* R,
                 bool sharded) {
  if (sharded) {
    double* w = c->dbuf("tsqr_work", tsqr_sharded_work_doubles(rows, s.l, s.comm->world));
    Comm* comm = s.comm;
    cudaStream_t st = c->st;
    launch_tsqr_sharded(X, s.lp, rows, s.l, s.lp, Q, s.lp, R, s.lp, w, s.flag, comm->world,
                        comm->rank,
                        [comm, st](const double* a, double* b, size_t n) { comm->allgather(a, b, n, st); },
                        st);
  } else {
    double* w = c->dbuf("tsqr_work", tsqr_work_doubles(rows, s.l));
    launch_tsqr(X, s.lp, rows, s.l, s.lp, Q, s.lp, R, s.lp, w, s.flag, c->st);
  }
}

void cholqr2(xb_ctx* c, const Small& s, const double* X, int64_t rows, double* T, double* Q,
             double* Rout, bool sharded = false) {
  const int l = s.l, lp = s.lp;
  cudaStream_t st = c->st;
  int* flag = s.flag;
  XB_CUDA(cudaMemsetAsync(s.flag, 0, sizeof(int), st));
  gram(c, s, X, rows, sharded);                                // G1 = X^T X
  launch_chol_inv(s.G, lp, l, 1e-12, s.R1, s.R1i, lp, flag, s.cw, st);
  gemm(c, false, rows, lp, lp, X, lp, s.R1i, lp, T, lp, 2);    // T = X R1^-1 (R1^-1 upper)
  gram(c, s, T, rows, sharded);                                // G2 = T^T T
  launch_chol_inv(s.G, lp, l, 1e-4, s.R2, s.R2i, lp, flag, s.cw, st);
  gemm(c, false, rows, lp, lp, T, lp, s.R2i, lp, Q, lp, 2);    // Q = T R2^-1
  double* R = Rout ? Rout : s.Rs;
  if (Rout) gemm(c, false, lp, lp, lp, s.R2, lp, s.R1, lp, Rout, lp);  // R = R2 R1
  qr_fallback(c, s, X, rows, Q, R, sharded);  // runs only when a Cholesky flagged
}

// Single-pass CholQR for the orthonormalisations INSIDE the power iteration.
// There Q only has to be a well-conditioned basis of range(X) for the next
// product: one pass gives ||Q^T Q - I|| ~ u kappa(X)^2 while range(Q) equals
// range(X) to ~u kappa(X), the same range accuracy as Householder. The
// pivot threshold (1e-8 G_jj, i.e. kappa below ~1e4 per column) keeps that
// loss far below the 1e-8 subspace target; beyond it the Householder
// fallback runs. The range-finder's final QR and the QR of B^T (whose Q
// must be orthonormal to machine precision) use cholqr2.
void cholqr1(xb_ctx* c, const Small& s, const double* X, int64_t rows, double* Q,
             bool sharded = false, double* Rout = nullptr) {
  const int l = s.l, lp = s.lp;
  cudaStream_t st = c->st;
  int* flag = s.flag;
  XB_CUDA(cudaMemsetAsync(s.flag, 0, sizeof(int), st));
  gram(c, s, X, rows, sharded, s.oz);                          // G = X^T X
  launch_chol_inv(s.G, lp, l, 1e-8, s.R1, s.R1i, lp, flag, s.cw, st);
  gemm_big(c, s.oz, false, rows, lp, lp, X, lp, s.R1i, lp, Q, lp, 2);  // Q = X R^-1
  if (Rout)
    XB_CUDA(cudaMemcpyAsync(Rout, s.R1, (size_t)lp * lp * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
  qr_fallback(c, s, X, rows, Q, Rout ? Rout : s.Rs, sharded);
}

// power = "auto" (pipeline.py:295-372). The reference watches the raw
// products Y_q = (A A^T)^q A Omega: nu_q = ||Y_q||_F / sqrt(m l). Here every
// product is re-orthonormalised, so the raw product is carried as a small
// upper-triangular factor: Y_q(raw) = Y_q C_q e^{L_q}, with C_0 = I, and
// after the QRs Y_q = Q R_q, Z = Q_z R_z:
//     ||Y_q(raw)||_F = e^{L_q} ||R_q C_q||_F,
//     C_{q+1} = R_z (R_q C_q) / ||R_q C_q||_F,  L_{q+1} = L_q + ln ||R_q C_q||_F
// (the normalisation keeps C bounded; only nu ratios enter the rule).
struct AutoPower {
  bool on = false;
  int lp = 0;
  double* C = nullptr;   // lp x lp
  double* M = nullptr;   // R_q C_q, normalised in place
  double* Rq = nullptr;  // R of the current Y
  double* Rz = nullptr;  // R of the current Z
  double* nrm = nullptr; // device scalar ||R_q C_q||_F
  double L = 0.0, scale = 1.0;
  std::vector<double> nus;
  double prev_rho = 1.0;
};

// nu of the current Y (R in a.Rq); returns ln nu
double auto_nu(xb_ctx* c, AutoPower& a) {
  gemm(c, false, a.lp, a.lp, a.lp, a.Rq, a.lp, a.C, a.lp, a.M, a.lp);
  launch_frob_normalise(a.M, (int64_t)a.lp * a.lp, a.nrm, c->st);
  double h = 0.0;
  XB_CUDA(cudaMemcpyAsync(&h, a.nrm, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  XB_CUDA(cudaStreamSynchronize(c->st));
  const double lognu = a.L + std::log(h);
  a.nus.push_back(h > 0.0 ? std::exp(lognu) * a.scale : 0.0);
  a.L = lognu;
  return lognu;
}

struct RsvdOut {
  double* U;
  int64_t ldu;
  double* s;
  double* V;
  int64_t ldv;
};

void check_dims(int64_t m, int64_t n, int k, int p, int q) {
  XB_REQUIRE(m >= 1 && n >= 1, XB_ESHAPE, "empty matrix");
  XB_REQUIRE(k >= 1, XB_EVALUE, "rank must be at least 1, got " + std::to_string(k));
  XB_REQUIRE(p >= 0, XB_EVALUE, "oversample must be nonnegative, got " + std::to_string(p));
  XB_REQUIRE(q >= 0 || q == XB_POWER_AUTO, XB_EVALUE,
             "power must be nonnegative, got " + std::to_string(q));
  XB_REQUIRE((int64_t)k + p <= std::min(m, n), XB_ESHAPE,
             "rank " + std::to_string(k) + " (+" + std::to_string(p) +
                 " oversampling) exceeds min(" + std::to_string(m) + ", " + std::to_string(n) +
                 ")");
}

// Where a host-resident A comes from, band by band of rows. Either one
// contiguous row-major array (the unbudgeted reference matrix is a single
// tile) or the reference's tile grid itself, fetched tile by tile
// through caller callbacks (a StoredMatrix of many tiles, possibly budgeted
// or store-backed: pool.get / read_cell_dense, pool.py:397-418) — then A is
// never assembled in host memory, and bands follow the grid's row cuts.
struct HostSource {
  virtual ~HostSource() {}
  // rows of the band starting at row r0 (<= cap when possible)
  virtual int64_t band_rows(int64_t r0, int64_t cap) const = 0;
  // enqueue the H2D copy of rows [r0, r0 + rows) (one or more whole bands)
  // into dst (ld elements per row) on stream s
  virtual void copy_rows(void* dst, int64_t ld, int64_t r0, int64_t rows, cudaStream_t s) = 0;
  // every copy enqueued so far has completed: host memory may be released
  virtual void copies_done() {}
  virtual bool pinned() const { return false; }
  virtual bool staged() const { return false; }
  // called once before the first copy: `streamed` = A will be read q + 1
  // times by the out-of-core streamer, else once into HBM
  virtual void prepare(xb_ctx*, bool /*streamed*/, int64_t /*m*/) {}
};

// geometry of the pageable-host staging ring: 6 x 8 MiB slots (the ring stays
// in the host's last-level cache, so the DMA reads it from there) filled in
// 256 KiB pieces (profiles/r02_stage_probe.md: 8.6 GB in 0.165-0.175 s against
// 0.155 s from pinned memory and 0.52 s with cudaHostRegister per call)
int knob_int(const char* name, int dflt) {
  const char* e = knob(name);
  return e && atoi(e) > 0 ? atoi(e) : dflt;
}
size_t stage_slot_bytes() {
  static const size_t v = (size_t)knob_int("XB_STAGE_SLOT_MB", 8) << 20;
  return v;
}
int stage_slots() {
  static const int v = knob_int("XB_STAGE_SLOTS", 6);
  return v;
}
size_t stage_piece_bytes() {
  static const size_t v = (size_t)knob_int("XB_STAGE_PIECE_KB", 256) << 10;
  return v;
}
// worker threads of the pageable-host staging ring
int stage_threads() {
  static const int n = [] {
    const char* e = knob("XB_STAGE_THREADS");
    if (e && atoi(e) > 0) return std::min(64, atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    // one core left to the thread that feeds the DMA queue
    return (int)std::max(2u, std::min(16u, hc ? hc : 8u) - 1u);
  }();
  return n;
}

struct ContiguousSource final : HostSource {
  const char* host;
  int64_t host_ld, n;
  size_t es;
  xb_ctx* ctx = nullptr;
  bool is_pinned_ = false, stage = false;
  void* registered = nullptr;
  ContiguousSource(const void* a, int64_t lda, int64_t cols, size_t esz)
      : host(static_cast<const char*>(a)), host_ld(lda), n(cols), es(esz) {
    is_pinned_ = is_pinned(host);
  }
  ~ContiguousSource() override {
    if (registered) cudaHostUnregister(registered);
  }
  // A pageable source goes through the staging ring, for the single in-HBM
  // ingest and for every pass of the out-of-core streamer alike: page-locking
  // runs at ~23 GB/s and has to be undone, the ring at ~50 GB/s per pass, so
  // registering would only pay beyond ~20 passes over A. Rows wider than a
  // slot are page-locked for the call instead; small inputs use pageable
  // copies.
  void prepare(xb_ctx* c, bool /*streamed*/, int64_t m) override {
    if (is_pinned_ || m <= 0) return;
    const size_t bytes = (size_t)((m - 1) * host_ld + n) * es;
    if (bytes < ((size_t)32 << 20)) return;
    const size_t slot_bytes = std::max<size_t>(stage_slot_bytes(), (size_t)round_up((int64_t)((size_t)n * es), 4096));
    if ((size_t)n * es > HostStager::kMaxRow) {
      if (cudaHostRegister(const_cast<char*>(host), bytes, cudaHostRegisterDefault) ==
          cudaSuccess) {
        registered = const_cast<char*>(host);
        is_pinned_ = true;
      } else {
        cudaGetLastError();  // pageable copies
      }
      return;
    }
    if (c->stager && c->stager->kSlot < slot_bytes) {
      delete c->stager;
      c->stager = nullptr;
    }
    if (!c->stager)
      c->stager = new HostStager(stage_threads(), stage_slots(), slot_bytes, stage_piece_bytes());
    ctx = c;
    stage = true;
  }
  int64_t band_rows(int64_t, int64_t cap) const override { return cap; }
  void copy_rows(void* dst, int64_t ld, int64_t r0, int64_t rows, cudaStream_t s) override {
    const char* src = host + (size_t)r0 * host_ld * es;
    if (stage)
      ctx->stager->copy(static_cast<char*>(dst), (size_t)ld * es, src, (size_t)host_ld * es,
                        (size_t)n * es, rows, s);
    else if (host_ld == n && ld == n)  // contiguous rows: one linear DMA
      XB_CUDA(cudaMemcpyAsync(dst, src, (size_t)rows * n * es, cudaMemcpyHostToDevice, s));
    else
      XB_CUDA(cudaMemcpy2DAsync(dst, ld * es, src, host_ld * es, n * es, rows,
                                cudaMemcpyHostToDevice, s));
  }
  bool pinned() const override { return is_pinned_; }
  bool staged() const override { return stage; }
};

struct TileSource final : HostSource {
  std::vector<int64_t> rcut, ccut;
  xb_tile_fetch_fn fetch;
  xb_tile_release_fn release;
  void* user;
  size_t es;
  std::vector<std::pair<int64_t, int64_t>> held;  // fetched, not yet released
  TileSource(const int64_t* row_cuts, int ntr, const int64_t* col_cuts, int ntc,
             xb_tile_fetch_fn f, xb_tile_release_fn r, void* u, size_t esz)
      : rcut(row_cuts, row_cuts + ntr + 1), ccut(col_cuts, col_cuts + ntc + 1), fetch(f),
        release(r), user(u), es(esz) {}
  ~TileSource() override { copies_done(); }
  int64_t band_index(int64_t r0) const {
    const auto it = std::upper_bound(rcut.begin(), rcut.end(), r0);
    return (int64_t)(it - rcut.begin()) - 1;
  }
  int64_t band_rows(int64_t r0, int64_t) const override {
    const int64_t ti = band_index(r0);
    return rcut[ti + 1] - r0;
  }
  void copy_rows(void* dst, int64_t ld, int64_t r0, int64_t rows, cudaStream_t s) override {
    for (int64_t r = r0; r < r0 + rows;) {
      const int64_t ti = band_index(r);
      XB_REQUIRE(rcut[ti] == r, XB_EVALUE, "tile source: copy not aligned to a row cut");
      const int64_t h = rcut[ti + 1] - rcut[ti];
      for (size_t tj = 0; tj + 1 < ccut.size(); ++tj) {
        int64_t tld = 0;
        const void* p = fetch(user, ti, (int64_t)tj, &tld);
        XB_REQUIRE(p != nullptr, XB_EVALUE,
                   "tile source: tile (" + std::to_string(ti) + ", " + std::to_string(tj) +
                       ") unavailable");
        held.push_back({ti, (int64_t)tj});
        const int64_t w = ccut[tj + 1] - ccut[tj];
        char* d = static_cast<char*>(dst) + ((size_t)(r - r0) * ld + ccut[tj]) * es;
        XB_CUDA(cudaMemcpy2DAsync(d, ld * es, p, tld * es, w * es, h, cudaMemcpyHostToDevice, s));
      }
      r += h;
    }
  }
  void copies_done() override {
    if (release)
      for (auto& t : held) release(user, t.first, t.second);
    held.clear();
  }
};

// Host-side description of how A reaches the device for the first product.
struct IngestPlan {
  HostSource* src = nullptr;  // non-null: stream row bands H2D, overlapped
  int64_t chunk_rows = 0;
};

// The operator A: dense (f64/f32, DMMA tile GEMM) or sparse (CSR of A and of
// A^T, gather SpMM). The reference dispatches the same way on density
// (kernels.py:79-112).
// Ozaki int8 slices of a dense f64 A, made once per factorisation: row
// slices for Y = A X and column slices of A^T for Z = A^T Q (ozgemm.cu).
struct OzA {
  int S = 0;  // 0: not sliced (DMMA path)
  int8_t* rows = nullptr;   // [S][kpn/32][mp][32]
  int32_t* erow = nullptr;  // m
  int64_t kpn = 0, mp = 0;
  int8_t* colsT = nullptr;  // [S][kpm/32][np][32]
  int32_t* ecol = nullptr;  // n
  int64_t kpm = 0, np = 0;
  // float32 A: digit slices made inside the GEMM (ozf_gemm); only the
  // row / column exponents are stored
  bool f32 = false;
};

struct AOp {
  bool sparse = false;
  OzA oz;
  AView dense{nullptr, 0, false};
  Csr csr, csrt;  // A (m x n) and A^T (n x m)
  // row-sharded A: this rank holds m local rows of an
  // m_global x n matrix; products over A^T and Grams of the m-side sketch
  // are summed over `comm`
  Comm* comm = nullptr;
  int64_t m_global = 0;
  // column-sharded A: this rank holds columns
  // [col0, col0 + n) of an m x n_global matrix; the products over A (Y = A X)
  // and the Grams of the n-side sketches are summed over `comm`, the m-side
  // QRs run replicated
  bool col_shard = false;
  int64_t n_global = 0, col0 = 0;
};

void spmm_on_a(xb_ctx* c, const Csr& s, const double* X, double* Y, int lp, int l) {
  cudaEvent_t b = nullptr, e = nullptr;
  if (c->profiling) {
    b = c->prof_event();
    e = c->prof_event();
    XB_CUDA(cudaEventRecord(b, c->st));
  }
  // Column panels: when the gathered operand is bigger than L2 but a
  // 64-column panel of it nearly fits (<= 110 MB: cfg3's 2e5 x 120 X), copy
  // each panel into a contiguous (cols x 64) buffer and run the gather SpMM
  // per panel — the gathers then hit L2 (83 % sector hits, 0.29-0.38 GB of
  // DRAM reads per panel instead of 11.9 GB per product), at the price of
  // one extra pass over A per panel. Measured at cfg3: step 44.6 -> 43.1 ms
  // with 64-column panels; 32-column panels (4 passes) 52.6 ms.
  // XB_SPMM_PANEL: -1 off, 0 auto, w forced.
  static const int panel_env = [] {
    const char* e = knob("XB_SPMM_PANEL");
    return e ? atoi(e) : 0;
  }();
  static const int blocks_env = [] {
    const char* e = knob("XB_SPMM_BLOCKS");
    return e ? atoi(e) : 0;
  }();
  int w = 0;
  if (panel_env > 0) {
    w = panel_env;
  } else if (panel_env == 0 && (double)s.cols * lp * 8.0 > 128e6) {
    if (64 < lp && (double)s.cols * 64 * 8.0 <= 110e6) w = 64;
  }
  if (w > 0 && w < lp) {
    double* P = c->dbuf("spmm_panel", (size_t)s.cols * w);
    for (int h0 = 0; h0 < lp; h0 += w) {
      const int wc = std::min(w, lp - h0);
      launch_copy2d(X + h0, s.cols, wc, lp, P, wc, c->st);
      launch_spmm(s, P, wc, Y + h0, lp, wc, c->st);
    }
  } else if (blocks_env >= 0 && (double)s.cols * lp * 8.0 > 256e6) {
    // Row blocks of the gathered operand: for A^T Q the 960 MB Q has no
    // L2-sized column panel, so A^T's segments (sorted by A row) are cut at
    // ~100 MB row blocks of Q and Z accumulates the blocks in order: every
    // pass gathers from one L2-sized window of Q (deterministic; the sum
    // order is block by block, each in row order). XB_SPMM_BLOCKS: -1 off,
    // 0 auto, n forced.
    const int nb = blocks_env > 0 ? blocks_env
                                  : (int)std::ceil((double)s.cols * lp * 8.0 / 100e6);
    const int64_t bw = ceil_div(s.cols, (int64_t)nb);
    int64_t* off = static_cast<int64_t*>(
        c->buf("spmm_off", (size_t)(nb + 1) * s.rows * sizeof(int64_t)));
    launch_seg_split(s, nb, bw, off, c->st);
    for (int b = 0; b < nb; ++b)
      launch_spmm_seg(s, off + (int64_t)b * s.rows, off + (int64_t)(b + 1) * s.rows, X, lp, Y, lp,
                      lp, b > 0, c->st);
  } else {
    launch_spmm(s, X, lp, Y, lp, lp, c->st);
  }
  if (c->profiling) {
    XB_CUDA(cudaEventRecord(e, c->st));
    // algorithmic bytes: 12 nnz + 8 (rows+1) + 8 l (cols_in + rows_out)
    const double bytes = 12.0 * s.nnz + 8.0 * (s.rows + 1) + 8.0 * l * (s.cols + s.rows);
    c->prof_pending.push_back({b, e, 2.0 * s.nnz * l, bytes, 0.0, 3});
  }
}

// Slice A once for the int8 tensor-core products (when the slices fit next
// to everything else in HBM); otherwise the products stay on DMMA.
// float32 A on the int8 pipe (ozf_gemm): exponents + range guard only;
// XB_F32_GEMM=tf32 keeps the 3xTF32 tcgen05 kernel.
bool ozf_enabled() {
  static const bool on = [] {
    const char* e = knob("XB_F32_GEMM");
    return !(e && (strcmp(e, "tf32") == 0 || strcmp(e, "dmma") == 0));
  }();
  return on;
}

void ozf_prepare(xb_ctx* c, AOp& op, int64_t m, int64_t n) {
  const AView& a = op.dense;
  if ((double)m * (double)n < (double)(1 << 24) || std::min(m, n) < 1024) return;
  if ((reinterpret_cast<uintptr_t>(a.p) & 15) != 0 || a.ld % 4 != 0) return;
  static const bool trace = getenv("XB_TRACE") != nullptr;
  OzA z;
  z.erow = c->ibuf("oz_erow", m);
  z.ecol = c->ibuf("oz_ecol", n);
  int* wide = c->ibuf("oz_wide", 1);
  void* scr = c->buf("oz_scr", oz_both_exp_scratch_bytes(m, n));
  XB_CUDA(cudaMemsetAsync(wide, 0, sizeof(int), c->st));
  oz_both_exp_f32(static_cast<const float*>(a.p), m, n, a.ld, z.erow, z.ecol, scr, wide, c->st);
  int hwide = 0;
  XB_CUDA(cudaMemcpyAsync(&hwide, wide, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  XB_CUDA(cudaStreamSynchronize(c->st));
  if (hwide) {
    if (trace) fprintf(stderr, "[xb] ozaki f32 off: dynamic-range guard\n");
    return;
  }
  if (trace) fprintf(stderr, "[xb] ozaki f32 on: 3 digit slices in the GEMM\n");
  z.S = 3;
  z.f32 = true;
  op.oz = z;
}

void oz_prepare(xb_ctx* c, AOp& op, int64_t m, int64_t n) {
  const AView& a = op.dense;
  if (op.sparse || !oz_enabled()) return;
  if (a.f32) {
    if (ozf_enabled()) ozf_prepare(c, op, m, n);
    return;
  }
  // small matrices stay on DMMA: slicing A costs ~1.5 passes over it and the
  // products are launch-bound (cfg1, 4096 x 2048: 1.2 ms DMMA vs 1.8 ms)
  if ((double)m * (double)n < (double)(1 << 24) || std::min(m, n) < 1024) return;
  const int64_t kpn = round_up(n, 32), kpm = round_up(m, 32);
  static const bool trace = getenv("XB_TRACE") != nullptr;
  OzA z;
  z.kpn = kpn;
  z.kpm = kpm;
  z.mp = round_up(m, 128);
  z.np = round_up(n, 128);
  z.erow = c->ibuf("oz_erow", m);
  z.ecol = c->ibuf("oz_ecol", n);
  int* wide = c->ibuf("oz_wide", 1);
  void* scr = c->buf("oz_scr", oz_both_exp_scratch_bytes(m, n));
  const double* A = static_cast<const double*>(a.p);
  // exponents + dynamic-range vote first (one small read-back per call):
  // 0 = every row/column within 64x its RMS (S digit slices), 1 = within
  // 16384x (one slice more keeps the same accuracy against the RMS scale),
  // 2 = wider: DMMA keeps f64 accuracy
  XB_CUDA(cudaMemsetAsync(wide, 0, sizeof(int), c->st));
  oz_both_exp(A, m, n, a.ld, z.erow, z.ecol, scr, wide, c->st);
  int hwide = 0;
  XB_CUDA(cudaMemcpyAsync(&hwide, wide, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  XB_CUDA(cudaStreamSynchronize(c->st));
  if (hwide >= 2) {
    if (trace) fprintf(stderr, "[xb] ozaki off: dynamic-range guard\n");
    return;
  }
  const int S = hwide == 1 ? std::max(7, oz_slices()) : oz_slices();
  z.S = S;
  const double need = (double)S * ((double)z.mp * kpn + (double)z.np * kpm);
  // slice buffers already cached at this size (a repeat call): no memory
  // query (a driver round trip on the hot path)
  const bool cached = c->buf_bytes("oz_rows") >= (size_t)S * z.mp * kpn &&
                      c->buf_bytes("oz_colsT") >= (size_t)S * z.np * kpm;
  size_t free_b = 0, total_b = 0;
  if (!cached && cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  const double have = (double)free_b + (double)c->cached_bytes();
  if (!cached && need + 2e9 > have) {
    if (trace) fprintf(stderr, "[xb] ozaki off: slices %.2f GB, free+cached %.2f GB\n", need / 1e9, have / 1e9);
    return;
  }
  if (trace) fprintf(stderr, "[xb] ozaki on: S=%d%s\n", S, hwide ? " (wide rows/columns)" : "");
  z.rows = static_cast<int8_t*>(c->buf("oz_rows", (size_t)S * z.mp * kpn));
  z.colsT = static_cast<int8_t*>(c->buf("oz_colsT", (size_t)S * z.np * kpm));
  oz_slice_both(A, m, n, a.ld, z.erow, z.ecol, z.rows, z.mp, kpn, z.colsT, z.np, kpm, S, c->st);
  op.oz = z;
}

// The right operand of one product over A (the f64 sketch X, K x lp),
// sliced once per product for the int8 paths: 3 digit planes for float32 A
// (ozf_gemm), S slices for the f64 slices of A (ozgemm).
struct RightOp {
  int32_t* ex = nullptr;
  int8_t* xs = nullptr;
  int64_t np = 0;
};

RightOp prep_right(xb_ctx* c, const AOp& op, bool tn, int64_t m, int64_t n, const double* X,
                   int lp) {
  RightOp r;
  if (op.sparse || (!op.oz.f32 && !op.oz.S)) return r;
  const int64_t Kk = tn ? m : n;
  auto* scr = static_cast<unsigned long long*>(c->buf("oz_xscr", (size_t)round_up(lp, 256) * 8));
  if (op.oz.f32) {
    r.np = round_up(lp, ozf_tile_n(lp));
    const int64_t kp = round_up(Kk, 32);
    r.ex = c->ibuf("ozf_ex", r.np);
    r.xs = static_cast<int8_t*>(c->buf("ozf_xs", (size_t)3 * r.np * kp));
    oz_col_exp(X, Kk, lp, lp, r.ex, scr, nullptr, c->st);
    oz_slice_right_f(X, Kk, lp, lp, r.ex, r.xs, r.np, kp, c->st);
  } else {
    r.np = round_up(lp, 64);
    const int64_t kp = tn ? op.oz.kpm : op.oz.kpn;
    r.ex = c->ibuf("oz_ex", r.np);
    r.xs = static_cast<int8_t*>(c->buf("oz_xs", (size_t)op.oz.S * r.np * kp));
    oz_col_exp(X, Kk, lp, lp, r.ex, scr, nullptr, c->st);
    oz_slice_right(X, Kk, lp, lp, r.ex, r.xs, r.np, kp, op.oz.S, c->st);
  }
  return r;
}

// Output rows [r0, r1) of one product over A: Y = A X (NN, rows of A) or
// Z = A^T Q (TN, columns of A), written to Y + r0 * lp. r0 is a multiple of
// 128 (the int8 slices' row tile) unless it is 0. Every kernel reads the
// sub-range through pointer offsets, with its original strides.
void product_rows(xb_ctx* c, const AOp& op, bool tn, int64_t m, int64_t n, const double* X,
                  double* Y, int lp, int l, const RightOp& ro, int64_t r0, int64_t r1) {
  if (r1 <= r0) return;
  const int64_t Kk = tn ? m : n, rows = r1 - r0;
  double* Yr = Y + r0 * lp;
  if (op.sparse) {
    Csr sub = tn ? op.csrt : op.csr;
    sub.rowptr += r0;
    sub.rows = rows;
    spmm_on_a(c, sub, X, Yr, lp, l);
    return;
  }
  if (!op.oz.f32 && !op.oz.S) {
    const AView& a = op.dense;
    const AView v{tn ? static_cast<const char*>(a.p) + (size_t)r0 * a.esz() : a.rows_from(r0), a.ld,
                  a.f32};
    gemm_on_a(c, tn, rows, lp, Kk, v, 0, X, lp, Yr, lp, l);
    return;
  }
  cudaEvent_t b = nullptr, e = nullptr;
  if (c->profiling) {
    b = c->prof_event();
    e = c->prof_event();
    XB_CUDA(cudaEventRecord(b, c->st));
  }
  const OzA& z = op.oz;
  if (z.f32) {
    const AView& a = op.dense;
    const float* A0 = static_cast<const float*>(a.p) + (tn ? r0 : r0 * a.ld);
    const size_t wd = ozf_workspace_doubles(rows, lp, Kk);
    double* work = wd ? c->dbuf("split", wd) : nullptr;
    ozf_gemm(A0, a.ld, tn, (tn ? z.ecol : z.erow) + r0, ro.xs, ro.np, ro.ex, rows, lp, Kk, Yr, lp,
             false, ozf_plan_splits(rows, lp, Kk), work, c->st);
  } else {
    const int64_t kp = tn ? z.kpm : z.kpn, rows_p = tn ? z.np : z.mp;
    const int8_t* L = (tn ? z.colsT : z.rows) + (size_t)(r0 / 128) * z.S * 128 * 32;
    const size_t wd = oz_workspace_doubles(rows, lp, Kk);
    double* work = wd ? c->dbuf("split", wd) : nullptr;
    ozgemm(L, rows_p, kp, (tn ? z.ecol : z.erow) + r0, ro.xs, ro.np, ro.ex, rows, lp, Kk, Yr, lp,
           false, z.S, work, c->st);
  }
  if (c->profiling) {
    XB_CUDA(cudaEventRecord(e, c->st));
    const double mn = (double)rows * (double)Kk;
    if (z.f32) {  // 6 int8 slice products over the padded tile grid
      const double ops = 6.0 * 2.0 * (double)round_up(rows, 128) * (double)ro.np *
                         (double)round_up(Kk, 32);
      c->prof_pending.push_back({b, e, 2.0 * mn * l, mn * 4.0, ops, 4});
    } else {  // S (S + 1) / 2 int8 slice products
      const double pairs = 0.5 * z.S * (z.S + 1);
      const double ops = pairs * 2.0 * (double)round_up(rows, 128) * (double)ro.np *
                         (double)(tn ? z.kpm : z.kpn);
      c->prof_pending.push_back({b, e, 2.0 * mn * l, mn * z.S, ops, 2});
    }
  }
}

// One product over A. Sharded products end in the one exchange of their
// layout (row shards: the n x l partials of A^T Q; column shards: the m x l
// partials of A X), overlapped with the product itself: the output rows are
// produced in chunks on the compute stream and each chunk's all-reduce runs
// on the communication stream while the next chunk computes.
void product(xb_ctx* c, const AOp& op, bool tn, int64_t m, int64_t n, const double* X,
             double* Y, int lp, int l, bool exchange) {
  const int64_t rows = tn ? n : m;
  const RightOp ro = prep_right(c, op, tn, m, n, X, lp);
  if (!exchange) {
    product_rows(c, op, tn, m, n, X, Y, lp, l, ro, 0, rows);
    return;
  }
  const int nch = rows >= 4 * 1024 ? 4 : 1;
  const int64_t step = nch > 1 ? round_up(ceil_div(rows, (int64_t)nch), 128) : rows;
  if (!c->cs) XB_CUDA(cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking));
  while ((int)c->xev.size() < 8) {
    cudaEvent_t ev;
    XB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->xev.push_back(ev);
  }
  int i = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += step, ++i) {
    const int64_t r1 = std::min(rows, r0 + step);
    product_rows(c, op, tn, m, n, X, Y, lp, l, ro, r0, r1);
    XB_CUDA(cudaEventRecord(c->xev[i % 4], c->st));
    XB_CUDA(cudaStreamWaitEvent(c->cs, c->xev[i % 4], 0));
    op.comm->allreduce_sum(Y + r0 * lp, (size_t)(r1 - r0) * lp, c->cs);
  }
  XB_CUDA(cudaEventRecord(c->xev[4], c->cs));
  XB_CUDA(cudaStreamWaitEvent(c->st, c->xev[4], 0));
}

// Y (m x lp) = A X
void op_nn(xb_ctx* c, const AOp& op, int64_t m, int64_t n, const double* X, double* Y, int lp,
           int l) {
  // column-sharded: Y = sum_g A_g X_g, the one m x l exchange per product
  product(c, op, false, m, n, X, Y, lp, l, op.comm && op.col_shard);
}

// Z (n x lp) = A^T Q
void op_tn(xb_ctx* c, const AOp& op, int64_t m, int64_t n, const double* Q, double* Z, int lp,
           int l) {
  // row-sharded: Z = sum_g A_g^T Q_g, the one n x l exchange per product
  product(c, op, true, m, n, Q, Z, lp, l, op.comm && !op.col_shard);
}

// One factorisation. A (device, f64 or f32 dense, or f64 CSR) is only touched
// by the products over A; everything downstream of a product is f64. With an
// f32 A, Omega is rounded through float32 first, as the reference stores it
// at the storage dtype (pipeline.py:281-282).
void rsvd_impl(xb_ctx* c, const AOp& op_in, int64_t m, int64_t n, const void* d_omega,
               int64_t ld_omega, uint64_t seed, int k, int p, int q, const RsvdOut& out,
               int32_t* deficient, int* ndeficient, double* stage_seconds, const IngestPlan& ing) {
  AOp op = op_in;
  const AView& a = op.dense;
  // m = rows held here (all of A unless row-sharded), n = columns held here
  // (all unless column-sharded)
  const bool sharded = op.comm != nullptr && !op.col_shard;  // m-side sums
  const bool csharded = op.comm != nullptr && op.col_shard;  // n-side sums
  check_dims(sharded ? op.m_global : m, csharded ? op.n_global : n, k, p, q);
  const int l = k + p;
  const int lp = (int)round_up(l, 8);
  const int kp = (int)round_up(k, 2);
  cudaStream_t st = c->st;
  StageClock clk(c);
  double local_stage[XB_NUM_STAGES] = {0};

  // workspaces (cached across calls)
  double* Om = c->dbuf("Om", (size_t)n * lp);
  double* Ym = c->dbuf("Ym", (size_t)m * lp);
  double* Tm = c->dbuf("Tm", (size_t)m * lp);
  double* Qm = c->dbuf("Qm", (size_t)m * lp);
  double* Zn = c->dbuf("Zn", (size_t)n * lp);
  double* Tn = c->dbuf("Tn", (size_t)n * lp);
  double* Qn = c->dbuf("Qn", (size_t)n * lp);
  double* Rf = c->dbuf("Rf", (size_t)lp * lp);
  double* Ub = c->dbuf("Ub", (size_t)lp * lp);
  double* Wk = c->dbuf("Wk", (size_t)lp * kp);
  double* sv = c->dbuf("sv", (size_t)lp);
  double* jw = c->dbuf("jw", jacobi_work_doubles(lp));
  int* jstat = c->ibuf("jstat", 4);
  int* defc = c->ibuf("defc", (size_t)lp + 4);
  // pre-size the split-K workspace for the largest product so no cudaMalloc
  // lands inside the timed stream
  {
    size_t need = 0;
    auto upd = [&](bool ta, int64_t M, int64_t N, int64_t K, bool af32) {
      DGemmArgs g{ta, M, N, K, nullptr, 0, nullptr, 0, nullptr, 0, af32};
      need = std::max(need, dgemm_workspace_doubles(g, dgemm_plan_splits(g)));
    };
    upd(false, m, lp, n, a.f32);
    upd(true, n, lp, m, a.f32);
    upd(true, lp, lp, m, false);
    upd(true, lp, lp, n, false);
    upd(false, m, lp, lp, false);
    upd(false, n, lp, lp, false);
    upd(false, m, k, lp, false);
    upd(false, n, k, lp, false);
    if (ing.src) upd(false, ing.chunk_rows, lp, n, a.f32);
    if (need) c->dbuf("split", need);
    // the TSQR fallback's workspace, so no allocation lands mid-stream
    c->dbuf("tsqr_work", op_in.comm ? tsqr_sharded_work_doubles(std::max(m, n), l, op_in.comm->world)
                                    : tsqr_work_doubles(std::max(m, n), l));
  }
  Small s = small_bufs(c, l);
  {
    static const bool qr_oz = [] {
      const char* e = knob("XB_QR_OZ");
      return !(e && atoi(e) == 0);
    }();
    s.oz = qr_oz && a.f32 && !op.sparse;
  }
  if (op.comm) s.comm = op.comm;
  XB_CUDA(cudaMemsetAsync(Ub, 0, (size_t)lp * lp * sizeof(double), st));
  XB_CUDA(cudaMemsetAsync(Wk, 0, (size_t)lp * kp * sizeof(double), st));

  // Preparation of O
  clk.enter(kGaussian);
  if (d_omega) {
    XB_CUDA(cudaMemsetAsync(Om, 0, (size_t)n * lp * sizeof(double), st));
    if (a.f32)
      launch_copy2d_cast<float, double>(static_cast<const float*>(d_omega), n, l, ld_omega, Om, lp,
                                        st);
    else
      launch_copy2d(static_cast<const double*>(d_omega), n, l, ld_omega, Om, lp, st);
  } else {
    // this rank's rows of Omega when column-sharded (rows are keyed by index)
    launch_gaussian<double>(seed, csharded ? op.col0 : 0, n, l, Om, lp, lp, st);
    if (a.f32) launch_round_f32(Om, n, l, lp, st);
  }

  // O*A^T: the sketch; with a host A, row chunks arrive on the copy stream and
  // each chunk's rows of Y are computed as soon as it lands.
  clk.enter(kSketch);
  if (ing.src) {
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    XB_CUDA(cudaEventCreate(&t0));
    XB_CUDA(cudaEventCreate(&t1));
    XB_CUDA(cudaEventRecord(t0, c->cp));
    std::vector<cudaEvent_t> landed;
    for (int64_t r0 = 0; r0 < m;) {
      const int64_t rows = std::min(ing.src->band_rows(r0, ing.chunk_rows), m - r0);
      ing.src->copy_rows(const_cast<void*>(a.rows_from(r0)), a.ld, r0, rows, c->cp);
      cudaEvent_t e;
      XB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      XB_CUDA(cudaEventRecord(e, c->cp));
      XB_CUDA(cudaStreamWaitEvent(st, e, 0));
      landed.push_back(e);
      gemm_on_a(c, false, rows, lp, n, a, r0, Om, lp, Ym + r0 * lp, lp, l);
      r0 += rows;
    }
    XB_CUDA(cudaEventRecord(t1, c->cp));
    XB_CUDA(cudaStreamSynchronize(c->cp));
    ing.src->copies_done();
    float ms = 0.f;
    XB_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    if (getenv("XB_TRACE"))
      fprintf(stderr, "[xb] ingest: %lld chunks, host pinned %d staged %d, %.1f ms (%.1f GB/s)\n",
              (long long)landed.size(), (int)ing.src->pinned(), (int)ing.src->staged(), ms,
              (double)m * n * a.esz() / (ms * 1e-3) / 1e9);
    local_stage[kParse] += ms * 1e-3;  // ingest (H2D), overlapped with the sketch
    for (auto e : landed) cudaEventDestroy(e);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    oz_prepare(c, op, m, n);  // the remaining products on the int8 slices
  } else {
    oz_prepare(c, op, m, n);
    op_nn(c, op, m, n, Om, Ym, lp, l);
  }
  // intermediate QRs (a basis for the next product) are single-pass, the
  // final range-finder QR is CholQR2 (see cholqr1)
  // (row-sharded: the m-side QRs sum their Grams over ranks; the n-side ones
  // run replicated on the all-reduced Z, identically on every rank)
  clk.enter(kOrtho);
  const bool autoq = q == XB_POWER_AUTO;
  const int qlim = autoq ? c->auto_qmax : q;
  AutoPower ap;
  if (autoq) {
    ap.on = true;
    ap.lp = lp;
    const size_t ll = (size_t)lp * lp;
    ap.C = c->dbuf("ap_C", ll);
    ap.M = c->dbuf("ap_M", ll);
    ap.Rq = c->dbuf("ap_Rq", ll);
    ap.Rz = c->dbuf("ap_Rz", ll);
    ap.nrm = c->dbuf("ap_nrm", 1);
    launch_identity(ap.C, lp, lp, st);
    ap.scale = 1.0 / std::sqrt((double)(op.comm ? op.m_global : m) * (double)l);
  }
  bool final_done = false, stop = false;
  int chosen = 0;
  double ln0 = 0.0, lnprev = 0.0;
  if (qlim == 0) {
    cholqr2(c, s, Ym, m, Tm, Qm, Rf, sharded);
    final_done = true;
  } else {
    cholqr1(c, s, Ym, m, Qm, sharded, autoq ? ap.Rq : nullptr);
  }
  if (autoq) {
    // the reference measures nu_0 even when q_max = 0 (R is then Rf)
    if (final_done) ap.Rq = Rf;
    ln0 = lnprev = auto_nu(c, ap);
    if (!(ap.nus[0] > 0.0)) stop = true;  // zero sketch: nothing to sharpen
  }
  for (int it = 0; it < qlim && !stop; ++it) {
    clk.enter(kSketch);
    op_tn(c, op, m, n, Qm, Zn, lp, l);  // Z = A^T Q
    clk.enter(kOrtho);
    cholqr1(c, s, Zn, n, Qn, csharded, autoq ? ap.Rz : nullptr);
    if (autoq) gemm(c, false, lp, lp, lp, ap.Rz, lp, ap.M, lp, ap.C, lp);  // C = R_z M
    clk.enter(kSketch);
    op_nn(c, op, m, n, Qn, Ym, lp, l);  // Y = A Qz
    clk.enter(kOrtho);
    chosen = it + 1;
    if (!autoq && it == q - 1) {
      cholqr2(c, s, Ym, m, Tm, Qm, Rf, sharded);
      final_done = true;
    } else {
      cholqr1(c, s, Ym, m, Qm, sharded, autoq ? ap.Rq : nullptr);
      if (autoq) {
        // stopping rule of pipeline.py:361-370
        const double ln = auto_nu(c, ap);
        if (ln < std::log(c->auto_tau) + ln0) {
          stop = true;
        } else {
          const double rho = std::exp(ln - lnprev);
          if (std::fabs(rho - ap.prev_rho) <= 0.01 * rho) stop = true;
          ap.prev_rho = rho;
        }
        lnprev = ln;
      }
    }
  }
  if (!final_done) cholqr2(c, s, Ym, m, Tm, Qm, Rf, sharded);  // the range basis: CholQR2
  c->last_q = autoq ? chosen : q;
  c->last_nus = ap.nus;
  // deficient columns of the final range-finder QR (kernels.py:327-331)
  launch_deficient(Rf, lp, l, a.f32 ? (double)FLT_EPSILON : DBL_EPSILON, defc, defc + 1, st);

  clk.enter(kProject);
  op_tn(c, op, m, n, Qm, Zn, lp, l);  // B^T = A^T Q
  if (c->gram_path) {
    // gram_path (pipeline.py:526-580): B^T of the power matrix,
    // (Q^T (A A^T)^q A)^T, as 2q thin products (raw, as the reference), then
    // the l x l Gram G = B B^T, its SVD (= eigen-decomposition, Jacobi on the
    // symmetric G), sigma = sqrt(eig)^(1/(2q+1)), V = B^T U_B with unit
    // columns, U = Q U_B.
    const int qg = c->last_q;
    for (int i = 0; i < qg; ++i) {
      op_nn(c, op, m, n, Zn, Tm, lp, l);  // A B^T
      op_tn(c, op, m, n, Tm, Zn, lp, l);  // A^T (A B^T)
    }
    clk.enter(kSvdPrep);
    gemm(c, true, lp, lp, n, Zn, lp, Zn, lp, s.G, lp);  // full G (Jacobi reads all of it)
    if (csharded) s.comm->allreduce_sum(s.G, (size_t)lp * lp, st);
    clk.enter(kSvd);
    launch_jacobi_svd(s.G, lp, l, k, Ub, lp, sv, Wk, kp, jw, jstat, st);
    launch_gram_sigma(sv, l, qg > 0 ? 1.0 / (2 * qg + 1) : 1.0, st);
    clk.enter(kPost);
    gemm(c, false, m, k, lp, Qm, lp, Ub, lp, out.U, out.ldu);    // U = Q U_B[:, :k]
    gemm(c, false, n, k, lp, Zn, lp, Ub, lp, out.V, out.ldv);    // V = B^T U_B[:, :k]
    gemm(c, true, k, k, n, out.V, out.ldv, out.V, out.ldv, s.Rs, k);  // column norms^2
    if (csharded) s.comm->allreduce_sum(s.Rs, (size_t)k * k, st);
    launch_scale_cols_by_diag(out.V, out.ldv, n, k, s.Rs, k, st);
  } else {

  clk.enter(kSvdPrep);
  // float32 configs: ONE CholQR pass of B^T and Q_B is never formed,
  // V = B^T (R_B^-1 W_k). Q_B's orthogonality loss u kappa(B)^2 (~1e-11 at
  // cfg5's kappa ~ 550) is far below the f32 target (1e-3 angle), and R_B
  // from the f64 Gram carries sigma to u kappa. float64 keeps CholQR2.
  const bool fused_lift = a.f32;
  double* lift = nullptr;
  if (fused_lift) {
    XB_CUDA(cudaMemsetAsync(s.flag, 0, sizeof(int), st));
    gram(c, s, Zn, n, csharded, s.oz);
    launch_chol_inv(s.G, lp, l, 1e-8, Rf, s.R1i, lp, s.flag, s.cw, st);
    // Cholesky breakdown: the TSQR Q replaces B^T in place, R^-1 := I
    qr_fallback(c, s, Zn, n, Zn, Rf, csharded);
    launch_identity_if(s.R1i, lp, l, s.flag, st);
  } else {
    cholqr2(c, s, Zn, n, Tn, Qn, Rf, csharded);  // B^T = Q_B R_B
  }

  clk.enter(kSvd);
  launch_jacobi_svd(Rf, lp, l, k, Ub, lp, sv, Wk, kp, jw, jstat, st, jacobi_tol(a.f32));

  clk.enter(kPost);
  gemm(c, false, m, k, lp, Qm, lp, Ub, lp, out.U, out.ldu);  // U = Q U_B[:, :k]
  if (fused_lift) {
    lift = c->dbuf("lift", (size_t)lp * kp);
    gemm(c, false, lp, kp, lp, s.R1i, lp, Wk, kp, lift, kp);   // R_B^-1 W_k
    gemm_big(c, s.oz, false, n, k, lp, Zn, lp, lift, kp, out.V, out.ldv);  // V = B^T R_B^-1 W_k
  } else {
    gemm(c, false, n, k, lp, Qn, lp, Wk, kp, out.V, out.ldv);  // V = Q_B W_k
  }
  }
  XB_CUDA(cudaMemcpyAsync(out.s, sv, k * sizeof(double), cudaMemcpyDeviceToDevice, st));

  int hstat = 0;
  std::vector<int> hdef(lp + 1, 0);
  XB_CUDA(cudaMemcpyAsync(&hstat, jstat, sizeof(int), cudaMemcpyDeviceToHost, st));
  XB_CUDA(cudaMemcpyAsync(hdef.data(), defc, (lp + 1) * sizeof(int), cudaMemcpyDeviceToHost, st));
  clk.finish(stage_seconds ? local_stage : nullptr);
  XB_CUDA(cudaStreamSynchronize(st));
  if (c->profiling) c->prof_collect();
  if (stage_seconds)
    for (int i = 0; i < XB_NUM_STAGES; ++i) stage_seconds[i] = local_stage[i];
  if (ndeficient) *ndeficient = hdef[0];
  if (deficient)
    for (int i = 0; i < hdef[0] && i < l; ++i) deficient[i] = hdef[1 + i];
  XB_REQUIRE(hstat == 0, XB_ECONV, "Jacobi SVD of the projected factor did not converge in 60 sweeps");
}

// ---- out-of-core: the pinned-host tile streamer (S1) ---------------------------
//
// Replaces the reference's residency machinery for matrices larger than
// memory (BlockPool LRU + spill lane, pool.py:189-221, 397-418) for the case
// A exceeds HBM (config 4: 256 GiB f32). A stays in (pinned) host memory and
// streams through HBM in row tiles, NB-deep on the copy stream, each tile's
// compute overlapping the next tiles' DMA. Every pass over A is fused
// (SURVEY §7 "cfg4 PCIe-bound passes"): with X the current basis,
//     Y_i = A_i X        and        W += A_i^T Y_i        (tile by tile)
// so one read of A yields both Y = A X and W = A^T Y. After the pass,
// CholQR of Y (resident in HBM) gives R, and A^T Q = W R^-1 — the next Z, or
// B^T after the last pass — without reading A again: q + 1 host passes
// instead of 2q + 2. If a Cholesky breaks down (R unusable), Z = A^T Q is
// recomputed with one extra TN-only pass.
struct Streamer {
  xb_ctx* c;
  HostSource* src;
  bool f32;
  int64_t m, n, tile_rows;  // tile_rows: the largest band
  static constexpr int NB = 3;
  void* tiles[NB];
  cudaEvent_t landed[NB], freed[NB], t0, t1;
  double copy_seconds = 0.0;
  size_t es() const { return f32 ? 4 : 8; }

  Streamer(xb_ctx* ctx, HostSource* source, bool is_f32, int64_t rows, int64_t cols,
           int64_t trows)
      : c(ctx), src(source), f32(is_f32), m(rows), n(cols), tile_rows(trows) {
    for (int b = 0; b < NB; ++b) {
      tiles[b] = c->buf("stream_tile" + std::to_string(b), (size_t)tile_rows * n * es());
      XB_CUDA(cudaEventCreateWithFlags(&landed[b], cudaEventDisableTiming));
      XB_CUDA(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
    }
    XB_CUDA(cudaEventCreate(&t0));
    XB_CUDA(cudaEventCreate(&t1));
  }
  ~Streamer() {
    for (int b = 0; b < NB; ++b) {
      cudaEventDestroy(landed[b]);
      cudaEventDestroy(freed[b]);
    }
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
  }

  // Stream all row bands; body(tile_view, r0, rows) enqueues the compute on
  // c->st for one band.
  template <typename F>
  void pass(F&& body) {
    XB_CUDA(cudaEventRecord(t0, c->cp));
    int64_t i = 0;
    for (int64_t r0 = 0; r0 < m; ++i) {
      const int b = (int)(i % NB);
      const int64_t rows = std::min(src->band_rows(r0, tile_rows), m - r0);
      XB_REQUIRE(rows <= tile_rows, XB_EVALUE, "streamer: band taller than its buffers");
      if (i >= NB) XB_CUDA(cudaStreamWaitEvent(c->cp, freed[b], 0));
      src->copy_rows(tiles[b], n, r0, rows, c->cp);
      XB_CUDA(cudaEventRecord(landed[b], c->cp));
      XB_CUDA(cudaStreamWaitEvent(c->st, landed[b], 0));
      body(AView{tiles[b], n, f32}, r0, rows);
      XB_CUDA(cudaEventRecord(freed[b], c->st));
      r0 += rows;
    }
    XB_CUDA(cudaEventRecord(t1, c->cp));
    XB_CUDA(cudaEventSynchronize(t1));
    src->copies_done();
    float ms = 0.f;
    XB_CUDA(cudaEventElapsedTime(&ms, t0, t1));
    copy_seconds += ms * 1e-3;
  }
};

// W (+)= tile^T Y_tile with the fixed tile order (deterministic sums).
void tn_accumulate(xb_ctx* c, const AView& t, int64_t rows, int64_t n, const double* Y, double* W,
                   int lp, int l) {
  cudaEvent_t b = nullptr, e = nullptr;
  if (c->profiling) {
    b = c->prof_event();
    e = c->prof_event();
    XB_CUDA(cudaEventRecord(b, c->st));
  }
  DGemmArgs g{true, n, lp, rows, t.p, t.ld, Y, lp, W, lp, t.f32, true};
  run_gemm(c, g);
  if (c->profiling) {
    XB_CUDA(cudaEventRecord(e, c->st));
    const double mn = (double)rows * n;
    const bool tg = tgemm_supported(g);
    c->prof_pending.push_back(
        {b, e, 2.0 * mn * l, mn * t.esz(), (tg ? 3.0 : 1.0) * 2.0 * mn * lp, tg ? 1 : 0});
  }
}

int host_flag(xb_ctx* c, const int* dflag) {
  int h = 0;
  XB_CUDA(cudaMemcpyAsync(&h, dflag, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  XB_CUDA(cudaStreamSynchronize(c->st));
  return h;
}

void rsvd_stream(xb_ctx* c, HostSource* hsrc, bool f32, int64_t m, int64_t n,
                 int64_t tile_rows, uint64_t seed, int k, int p, int q, const RsvdOut& out,
                 int32_t* deficient, int* ndeficient, double* stage_seconds) {
  check_dims(m, n, k, p, q);
  const int l = k + p;
  const int lp = (int)round_up(l, 8);
  const int kp = (int)round_up(k, 2);
  cudaStream_t st = c->st;
  StageClock clk(c);
  double local_stage[XB_NUM_STAGES] = {0};
  double* Om = c->dbuf("Om", (size_t)n * lp);
  double* Ym = c->dbuf("Ym", (size_t)m * lp);
  double* Tm = c->dbuf("Tm", (size_t)m * lp);
  double* Qm = c->dbuf("Qm", (size_t)m * lp);
  double* Wn = c->dbuf("Wn", (size_t)n * lp);
  double* Zn = c->dbuf("Zn", (size_t)n * lp);
  double* Tn = c->dbuf("Tn", (size_t)n * lp);
  double* Qn = c->dbuf("Qn", (size_t)n * lp);
  double* Rf = c->dbuf("Rf", (size_t)lp * lp);
  double* Ub = c->dbuf("Ub", (size_t)lp * lp);
  double* Wk = c->dbuf("Wk", (size_t)lp * kp);
  double* sv = c->dbuf("sv", (size_t)lp);
  double* jw = c->dbuf("jw", jacobi_work_doubles(lp));
  int* jstat = c->ibuf("jstat", 4);
  int* defc = c->ibuf("defc", (size_t)lp + 4);
  c->dbuf("tsqr_work", tsqr_work_doubles(std::max(m, n), l));
  {
    size_t need = 0;
    auto upd = [&](bool ta, int64_t M, int64_t N, int64_t K, bool af32) {
      DGemmArgs g{ta, M, N, K, nullptr, 0, nullptr, 0, nullptr, 0, af32};
      need = std::max(need, dgemm_workspace_doubles(g, dgemm_plan_splits(g)));
    };
    upd(false, tile_rows, lp, n, f32);
    upd(true, n, lp, tile_rows, f32);
    upd(true, lp, lp, m, false);
    upd(true, lp, lp, n, false);
    upd(false, m, lp, lp, false);
    upd(false, n, lp, lp, false);
    upd(false, m, k, lp, false);
    upd(false, n, k, lp, false);
    if (need) c->dbuf("split", need);
  }
  Streamer sm(c, hsrc, f32, m, n, tile_rows);
  Small s = small_bufs(c, l);
  XB_CUDA(cudaMemsetAsync(Ub, 0, (size_t)lp * lp * sizeof(double), st));
  XB_CUDA(cudaMemsetAsync(Wk, 0, (size_t)lp * kp * sizeof(double), st));

  clk.enter(kGaussian);
  launch_gaussian<double>(seed, 0, n, l, Om, lp, lp, st);
  if (f32) launch_round_f32(Om, n, l, lp, st);

  // one fused pass: Y = A X and W = A^T Y
  auto fused_pass = [&](const double* X) {
    XB_CUDA(cudaMemsetAsync(Wn, 0, (size_t)n * lp * sizeof(double), st));
    sm.pass([&](const AView& t, int64_t r0, int64_t rows) {
      gemm_on_a(c, false, rows, lp, n, t, 0, X, lp, Ym + r0 * lp, lp, l);
      tn_accumulate(c, t, rows, n, Ym + r0 * lp, Wn, lp, l);
    });
  };
  // fallback: Z = A^T Q directly (one TN-only pass)
  auto tn_pass = [&](const double* Q, double* Z) {
    XB_CUDA(cudaMemsetAsync(Z, 0, (size_t)n * lp * sizeof(double), st));
    sm.pass([&](const AView& t, int64_t r0, int64_t rows) {
      tn_accumulate(c, t, rows, n, Q + r0 * lp, Z, lp, l);
    });
  };

  // power = "auto" (pipeline.py:295-372): the same carried-R stopping rule
  // as rsvd_impl; every fused pass yields the raw Y of the next power, so
  // the rule costs no extra pass over A, and stopping after pass `it` finds
  // B^T = W R^-1 already in hand
  const bool autoq = q == XB_POWER_AUTO;
  const int qlim = autoq ? c->auto_qmax : q;
  AutoPower ap;
  if (autoq) {
    ap.on = true;
    ap.lp = lp;
    const size_t ll = (size_t)lp * lp;
    ap.C = c->dbuf("ap_C", ll);
    ap.M = c->dbuf("ap_M", ll);
    ap.Rq = c->dbuf("ap_Rq", ll);
    ap.Rz = c->dbuf("ap_Rz", ll);
    ap.nrm = c->dbuf("ap_nrm", 1);
    launch_identity(ap.C, lp, lp, st);
    ap.scale = 1.0 / std::sqrt((double)m * (double)l);
  }
  const double* X = Om;
  int chosen = 0;
  double ln0 = 0.0, lnprev = 0.0;
  for (int it = 0; it <= qlim; ++it) {
    clk.enter(kSketch);
    fused_pass(X);
    clk.enter(kOrtho);
    bool last = it == qlim;
    if (autoq) {
      cholqr1(c, s, Ym, m, Qm, false, ap.Rq);  // R of the raw-product chain
      const double ln = auto_nu(c, ap);
      if (it == 0) {
        ln0 = lnprev = ln;
        if (!(ap.nus[0] > 0.0)) last = true;  // zero sketch: nothing to sharpen
      } else {
        // stopping rule of pipeline.py:361-370
        if (ln < std::log(c->auto_tau) + ln0) {
          last = true;
        } else {
          const double rho = std::exp(ln - lnprev);
          if (std::fabs(rho - ap.prev_rho) <= 0.01 * rho) last = true;
          ap.prev_rho = rho;
        }
        lnprev = ln;
      }
    }
    if (!last) {
      if (!autoq) cholqr1(c, s, Ym, m, Qm);  // R^-1 in s.R1i unless the fallback ran
      clk.enter(kSketch);
      if (host_flag(c, s.flag))
        tn_pass(Qm, Zn);
      else
        gemm(c, false, n, lp, lp, Wn, lp, s.R1i, lp, Zn, lp);  // Z = W R^-1 = A^T Q
      clk.enter(kOrtho);
      cholqr1(c, s, Zn, n, Qn, false, autoq ? ap.Rz : nullptr);
      if (autoq) gemm(c, false, lp, lp, lp, ap.Rz, lp, ap.M, lp, ap.C, lp);  // C = R_z M
      X = Qn;
      chosen = it + 1;
    } else {
      cholqr2(c, s, Ym, m, Tm, Qm, Rf);
      clk.enter(kProject);
      if (host_flag(c, s.flag)) {
        tn_pass(Qm, Zn);  // B^T = A^T Q
      } else {
        gemm(c, false, n, lp, lp, Wn, lp, s.R1i, lp, Tn, lp);  // B^T = W R1^-1 R2^-1
        gemm(c, false, n, lp, lp, Tn, lp, s.R2i, lp, Zn, lp);
      }
      break;
    }
  }
  c->last_q = autoq ? chosen : q;
  c->last_nus = ap.nus;
  launch_deficient(Rf, lp, l, f32 ? (double)FLT_EPSILON : DBL_EPSILON, defc, defc + 1, st);
  if (c->gram_path) {
    // gram_path (pipeline.py:526-580): B^T of the power matrix by 2q raw
    // products — each a fused pass with X = B^T (Y' = A B^T, W = A^T Y') —
    // then the l x l Gram, its eigen-decomposition by Jacobi, sigma =
    // sqrt(eig)^(1/(2q+1)), U = Q U_B, V = B^T U_B with unit columns
    const int qg = c->last_q;
    for (int i = 0; i < qg; ++i) {
      clk.enter(kProject);
      fused_pass(Zn);
      XB_CUDA(cudaMemcpyAsync(Zn, Wn, (size_t)n * lp * sizeof(double), cudaMemcpyDeviceToDevice,
                              st));
    }
    clk.enter(kSvdPrep);
    gemm(c, true, lp, lp, n, Zn, lp, Zn, lp, s.G, lp);  // full G (Jacobi reads all of it)
    clk.enter(kSvd);
    launch_jacobi_svd(s.G, lp, l, k, Ub, lp, sv, Wk, kp, jw, jstat, st);
    launch_gram_sigma(sv, l, qg > 0 ? 1.0 / (2 * qg + 1) : 1.0, st);
    clk.enter(kPost);
    gemm(c, false, m, k, lp, Qm, lp, Ub, lp, out.U, out.ldu);  // U = Q U_B[:, :k]
    gemm(c, false, n, k, lp, Zn, lp, Ub, lp, out.V, out.ldv);  // V = B^T U_B[:, :k]
    gemm(c, true, k, k, n, out.V, out.ldv, out.V, out.ldv, s.Rs, k);  // column norms^2
    launch_scale_cols_by_diag(out.V, out.ldv, n, k, s.Rs, k, st);
  } else {
    clk.enter(kSvdPrep);
    cholqr2(c, s, Zn, n, Tn, Qn, Rf);
    clk.enter(kSvd);
    launch_jacobi_svd(Rf, lp, l, k, Ub, lp, sv, Wk, kp, jw, jstat, st, jacobi_tol(f32));
    clk.enter(kPost);
    gemm(c, false, m, k, lp, Qm, lp, Ub, lp, out.U, out.ldu);
    gemm(c, false, n, k, lp, Qn, lp, Wk, kp, out.V, out.ldv);
  }
  XB_CUDA(cudaMemcpyAsync(out.s, sv, k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int hstat = 0;
  std::vector<int> hdef(lp + 1, 0);
  XB_CUDA(cudaMemcpyAsync(&hstat, jstat, sizeof(int), cudaMemcpyDeviceToHost, st));
  XB_CUDA(cudaMemcpyAsync(hdef.data(), defc, (lp + 1) * sizeof(int), cudaMemcpyDeviceToHost, st));
  clk.finish(stage_seconds ? local_stage : nullptr);
  XB_CUDA(cudaStreamSynchronize(st));
  if (c->profiling) c->prof_collect();
  local_stage[kParse] += sm.copy_seconds;  // host->HBM streaming (overlapped with compute)
  if (stage_seconds)
    for (int i = 0; i < XB_NUM_STAGES; ++i) stage_seconds[i] = local_stage[i];
  if (ndeficient) *ndeficient = hdef[0];
  if (deficient)
    for (int i = 0; i < hdef[0] && i < l; ++i) deficient[i] = hdef[1 + i];
  XB_REQUIRE(hstat == 0, XB_ECONV, "Jacobi SVD of the projected factor did not converge in 60 sweeps");
}

int64_t auto_tile_rows(int64_t m, int64_t n, size_t es) {
  int64_t r = std::max<int64_t>(256, ((int64_t)1 << 31) / std::max<int64_t>(n * (int64_t)es, 1));
  r = r / 256 * 256;
  return std::max<int64_t>(1, std::min(r, m));
}

// Does A (m x n of `es` bytes) fit in HBM next to the factorisation's buffers?
// Does A fit in HBM next to the sketch buffers? This context's cached
// buffers count as available (buf() releases stale ones on demand).
bool fits_in_hbm(const xb_ctx* c, int64_t m, int64_t n, size_t es, int lp) {
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  free_b += c->cached_bytes();
  const double need = (double)m * n * es + (4.0 * m + 5.0 * n) * lp * 8.0 + 2.0 * 2 * std::max(m, n) * lp * 8.0 +
                      (double)(1ull << 30);
  return need < (double)free_b;
}

// true for float32 (Precision.SINGLE), false for float64
bool check_dtype(int dtype) {
  XB_REQUIRE(dtype == XB_F64 || dtype == XB_F32, XB_EVALUE, "unknown dtype");
  return dtype == XB_F32;
}

// C = op(A) B for device operands of one dtype. float32 follows the
// reference's storage rule (core.py:43-46: f32 in, f32 out) but accumulates
// in f64: A is widened in the kernel, B and C go through f64 scratch.
void gemm_any(xb_ctx* c, bool f32, bool ta, int64_t m, int64_t n, int64_t kdim, const void* dA,
              int64_t lda, const void* dB, int64_t ldb, void* dC, int64_t ldc) {
  if (!f32) {
    static const bool oz_dbg = knob("XB_GEMM_OZ") != nullptr;
    if (oz_dbg && m > 0 && n > 0 && kdim > 0) {
      // diagnostics (tools/oz_check.py): the same product on the int8 slices
      oz_gemm64(c, ta, m, n, kdim, static_cast<const double*>(dA), lda,
                static_cast<const double*>(dB), ldb, static_cast<double*>(dC), ldc, 0,
                oz_slices());
      return;
    }
    gemm(c, ta, m, n, kdim, static_cast<const double*>(dA), lda, static_cast<const double*>(dB),
         ldb, static_cast<double*>(dC), ldc);
    return;
  }
  const int64_t np = round_up(n, 2);
  double* B64 = c->dbuf("gB64", (size_t)std::max<int64_t>(1, kdim * np));
  double* C64 = c->dbuf("gC64", (size_t)m * np);
  launch_copy2d_cast<float, double>(static_cast<const float*>(dB), kdim, n, ldb, B64, np, c->st);
  static const bool ozf_dbg = knob("XB_GEMM_OZF") != nullptr;
  if (ozf_dbg && m > 0 && n > 0 && kdim > 0) {
    // diagnostics (tools/ozf_check.py): float32 A on the int8 pipe
    const float* A = static_cast<const float*>(dA);
    const int64_t rows = ta ? kdim : m, cols = ta ? m : kdim;
    int32_t* er = c->ibuf("dbg_er", rows);
    int32_t* ec = c->ibuf("dbg_ec", cols);
    void* scr = c->buf("dbg_rc", oz_both_exp_scratch_bytes(rows, cols));
    oz_both_exp_f32(A, rows, cols, lda, er, ec, scr, nullptr, c->st);
    const int64_t kp = round_up(kdim, 32), npf = round_up(n, ozf_tile_n(n));
    int32_t* eR = c->ibuf("dbg_eR", npf);
    auto* scr2 = static_cast<unsigned long long*>(c->buf("dbg_scr", (size_t)npf * 8));
    int8_t* R = static_cast<int8_t*>(c->buf("dbg_Rf", (size_t)3 * npf * kp));
    const size_t wd = ozf_workspace_doubles(m, n, kdim);
    double* work = wd ? c->dbuf("split", wd) : nullptr;
    oz_col_exp(B64, kdim, n, np, eR, scr2, nullptr, c->st);
    oz_slice_right_f(B64, kdim, n, np, eR, R, npf, kp, c->st);
    ozf_gemm(A, lda, ta, ta ? ec : er, R, npf, eR, m, n, kdim, C64, np, false,
             ozf_plan_splits(m, n, kdim), work, c->st);
    launch_copy2d_cast<double, float>(C64, m, n, np, static_cast<float*>(dC), ldc, c->st);
    return;
  }
  DGemmArgs g{ta, m, n, kdim, dA, lda, B64, np, C64, np, true};
  run_gemm(c, g);
  launch_copy2d_cast<double, float>(C64, m, n, np, static_cast<float*>(dC), ldc, c->st);
}

}  // namespace

// ---- C ABI ---------------------------------------------------------------------

extern "C" {

int xb_abi_version(void) { return XB_ABI_VERSION; }

int xb_build_flags(void) { return experiments_build() ? XB_BUILD_EXPERIMENTS : 0; }

const char* xb_last_error(void) { return g_last_error.c_str(); }

int xb_create(int device, xb_ctx** out) {
  return guarded([&] {
    XB_REQUIRE(out != nullptr, XB_EVALUE, "out is null");
    int n = 0;
    XB_CUDA(cudaGetDeviceCount(&n));
    XB_REQUIRE(device >= 0 && device < n, XB_EVALUE, "no such CUDA device");
    auto* c = new xb_ctx();
    c->device = device;
    XB_CUDA(cudaSetDevice(device));
    XB_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    XB_CUDA(cudaStreamCreateWithFlags(&c->cp, cudaStreamNonBlocking));
    *out = c;
  });
}

int xb_destroy(xb_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    cudaStreamSynchronize(c->cp);
    for (auto& kv : c->bufs) cudaFree(kv.second.p);
    for (auto e : c->events) cudaEventDestroy(e);
    delete c->stager;
    delete c->comm;
    if (c->cs) {
      cudaStreamSynchronize(c->cs);
      cudaStreamDestroy(c->cs);
    }
    for (auto e : c->xev) cudaEventDestroy(e);
    cudaStreamDestroy(c->st);
    cudaStreamDestroy(c->cp);
    if (c->caller_ev) cudaEventDestroy(c->caller_ev);
    delete c;
  });
}

int64_t xb_launch_count(const xb_ctx* c) { return c ? c->launches : 0; }

void* xb_compute_stream(xb_ctx* c) { return c ? static_cast<void*>(c->st) : nullptr; }

int xb_set_power_auto(xb_ctx* c, int q_max, double tau) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    XB_REQUIRE(q_max >= 0, XB_EVALUE, "q_max must be nonnegative, got " + std::to_string(q_max));
    XB_REQUIRE(tau > 0.0, XB_EVALUE, "tau must be positive");
    c->auto_qmax = q_max;
    c->auto_tau = tau;
  });
}

int xb_last_power(xb_ctx* c, int* chosen_q, double* nus, int cap, int* count) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    if (chosen_q) *chosen_q = c->last_q;
    const int nn = (int)c->last_nus.size();
    if (count) *count = nn;
    for (int i = 0; nus && i < nn && i < cap; ++i) nus[i] = c->last_nus[i];
  });
}

int xb_set_gram_path(xb_ctx* c, int on) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    c->gram_path = on != 0;
  });
}

int xb_profile_enable(xb_ctx* c, int on) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    c->profiling = on != 0;
  });
}

int xb_profile_read(xb_ctx* c, double* out4) {
  return guarded([&] {
    XB_REQUIRE(c && out4, XB_EVALUE, "null argument");
    XB_CUDA(cudaStreamSynchronize(c->st));
    c->prof_collect();
    for (int i = 0; i < 4; ++i) out4[i] = c->prof_acc[i];
    for (int i = 0; i < 6; ++i) c->prof_acc[i] = i == 5 ? -1.0 : 0.0;
  });
}

int xb_profile_read_ext(xb_ctx* c, double* out6) {
  return guarded([&] {
    XB_REQUIRE(c && out6, XB_EVALUE, "null argument");
    XB_CUDA(cudaStreamSynchronize(c->st));
    c->prof_collect();
    for (int i = 0; i < 6; ++i) {
      out6[i] = c->prof_acc[i];
      c->prof_acc[i] = i == 5 ? -1.0 : 0.0;
    }
  });
}

int xb_fp64_peaks(xb_ctx* c, double* dmma_tflops, double* dfma_tflops) {
  return guarded([&] {
    XB_REQUIRE(c && dmma_tflops && dfma_tflops, XB_EVALUE, "null argument");
    LaunchScope ls(c);
    measure_fp64_peaks(c->st, dmma_tflops, dfma_tflops);
  });
}

int xb_tc_peaks(xb_ctx* c, double* i8_tops, double* bf16_tflops) {
  return guarded([&] {
    XB_REQUIRE(c && i8_tops && bf16_tflops, XB_EVALUE, "null argument");
    LaunchScope ls(c);
    measure_tc_peaks(c->st, i8_tops, bf16_tflops, 0);
  });
}

int xb_tc_peaks_data(xb_ctx* c, int random_data, double* i8_tops, double* bf16_tflops) {
  return guarded([&] {
    XB_REQUIRE(c && i8_tops && bf16_tflops, XB_EVALUE, "null argument");
    LaunchScope ls(c);
    measure_tc_peaks(c->st, i8_tops, bf16_tflops, random_data != 0);
  });
}

int xb_rsvd_dense_dev(xb_ctx* c, int dtype, int64_t m, int64_t n, const void* dA, int64_t lda,
                      const void* d_omega, uint64_t seed, int k, int p, int q, void* dU,
                      int64_t ldu, double* d_s, void* dV, int64_t ldv, int32_t* deficient,
                      int* ndeficient, double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    after_caller_stream(c);
    const bool f32 = check_dtype(dtype);
    XB_REQUIRE(lda >= n && ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    AOp a;
    a.dense = AView{dA, lda, f32};
    if (!f32) {
      RsvdOut out{static_cast<double*>(dU), ldu, d_s, static_cast<double*>(dV), ldv};
      rsvd_impl(c, a, m, n, d_omega, k + p, seed, k, p, q, out, deficient, ndeficient,
                stage_seconds, IngestPlan{});
      return;
    }
    // float32 outputs: factors are formed in f64, then stored at the storage
    // dtype like the reference (pipeline.py:589-591, 603-611)
    double* Ud = c->dbuf("Ud", (size_t)m * k);
    double* Vd = c->dbuf("Vd", (size_t)n * k);
    RsvdOut out{Ud, k, d_s, Vd, k};
    rsvd_impl(c, a, m, n, d_omega, k + p, seed, k, p, q, out, deficient, ndeficient,
              stage_seconds, IngestPlan{});
    launch_copy2d_cast<double, float>(Ud, m, k, k, static_cast<float*>(dU), ldu, c->st);
    launch_copy2d_cast<double, float>(Vd, n, k, k, static_cast<float*>(dV), ldv, c->st);
    XB_CUDA(cudaStreamSynchronize(c->st));
  });
}

}  // extern "C"

namespace {

// First touch of the caller's pageable output arrays while the GPU computes:
// a fresh numpy result is untouched memory, and its first-touch page faults
// (serialised on the process's mmap lock) otherwise land inside the
// device -> host copy at the end of the call. One byte per 4 KiB page is
// written from a helper thread; the copies overwrite everything afterwards.
struct OutputPretouch {
  std::thread th;
  void add(std::vector<std::pair<char*, size_t>>& v, void* p, size_t ld_bytes, size_t row_bytes,
           int64_t rows) {
    if (!p || rows <= 0 || is_pinned(p)) return;
    const size_t span = (size_t)(rows - 1) * ld_bytes + row_bytes;
    if (span >= ((size_t)4 << 20) && ld_bytes == row_bytes) v.push_back({static_cast<char*>(p), span});
  }
  OutputPretouch(void* U, size_t ldu_b, size_t urow_b, int64_t m, void* V, size_t ldv_b,
                 size_t vrow_b, int64_t n) {
    std::vector<std::pair<char*, size_t>> spans;
    add(spans, U, ldu_b, urow_b, m);
    add(spans, V, ldv_b, vrow_b, n);
    if (spans.empty()) return;
    th = std::thread([spans] {
      for (auto& sp : spans) {
        volatile char* q = sp.first;
        for (size_t o = 0; o < sp.second; o += 4096) q[o] = 0;
        q[sp.second - 1] = 0;
      }
    });
  }
  void join() {
    if (th.joinable()) th.join();
  }
  ~OutputPretouch() { join(); }
};

// One factorisation of a host-resident dense A (any HostSource) with host
// outputs: in HBM when A fits next to the sketch buffers (bands ingested on
// the copy stream, each band's rows of the first product computed as it
// lands), else the out-of-core streamer (q + 1 fused passes over A).
void rsvd_from_host(xb_ctx* c, bool f32, int64_t m, int64_t n, HostSource& src,
                    int64_t max_band, bool force_stream, int64_t stream_rows, const void* omega,
                    uint64_t seed, int k, int p, int q, void* U, int64_t ldu, double* s, void* V,
                    int64_t ldv, int32_t* deficient, int* ndeficient, double* stage_seconds) {
  const size_t es = f32 ? 4 : 8;
  const int l = k + p;
  const double t0 = now_s();
  OutputPretouch touch(U, (size_t)ldu * es, (size_t)k * es, m, V, (size_t)ldv * es, (size_t)k * es, n);
  double* dU = c->dbuf("U", (size_t)m * k);
  double* dV = c->dbuf("V", (size_t)n * k);
  double* ds = c->dbuf("s", (size_t)k);
  RsvdOut out{dU, k, ds, dV, k};
  const int lp = (int)round_up(l, 8);
  const bool stream = force_stream || !fits_in_hbm(c, m, n, es, lp);
  src.prepare(c, stream, m);
  double t1 = 0.0;
  if (stream) {
    XB_REQUIRE(omega == nullptr, XB_EUNSUPPORTED,
               "an explicit Omega is not supported by the out-of-core streamer");
    int64_t tr = max_band > 0 ? max_band
                 : stream_rows > 0 ? std::min<int64_t>(stream_rows, m)
                                   : auto_tile_rows(m, n, es);
    t1 = now_s();
    rsvd_stream(c, &src, f32, m, n, tr, seed, k, p, q, out, deficient, ndeficient, stage_seconds);
  } else {
    void* dA = c->buf("A", (size_t)m * n * es);
    void* dO = nullptr;
    if (omega) {
      dO = c->buf("omega_in", (size_t)n * l * es);
      XB_CUDA(cudaMemcpyAsync(dO, omega, (size_t)n * l * es, cudaMemcpyHostToDevice, c->st));
    }
    IngestPlan ing;
    ing.src = &src;
    if (max_band > 0) {
      ing.chunk_rows = max_band;  // the tile grid's row bands
    } else {
      // ~1 GiB chunks, at least 8 of them when the matrix is large
      int64_t rows =
          std::max<int64_t>(256, ((int64_t)1 << 30) / std::max<int64_t>(n * (int64_t)es, 1));
      rows = std::min(rows, std::max<int64_t>(256, round_up(ceil_div(m, 8), 128)));
      ing.chunk_rows = std::min(rows, m);
    }
    t1 = now_s();
    AOp op;
    op.dense = AView{dA, n, f32};
    rsvd_impl(c, op, m, n, dO, l, seed, k, p, q, out, deficient, ndeficient, stage_seconds, ing);
  }
  const double t2 = now_s();
  void* oU = dU;
  void* oV = dV;
  if (f32) {
    oU = c->buf("U32", (size_t)m * k * 4);
    oV = c->buf("V32", (size_t)n * k * 4);
    launch_copy2d_cast<double, float>(dU, m, k, k, static_cast<float*>(oU), k, c->st);
    launch_copy2d_cast<double, float>(dV, n, k, k, static_cast<float*>(oV), k, c->st);
  }
  XB_CUDA(cudaMemcpyAsync(s, ds, k * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  touch.join();
  d2h_rows(c, U, ldu * es, oU, k * es, k * es, m);
  d2h_rows(c, V, ldv * es, oV, k * es, k * es, n);
  XB_CUDA(cudaStreamSynchronize(c->st));
  if (getenv("XB_TRACE"))
    fprintf(stderr, "[xb] rsvd host A: setup %.1f ms, ingest+compute %.1f ms, d2h %.1f ms\n",
            (t1 - t0) * 1e3, (t2 - t1) * 1e3, (now_s() - t2) * 1e3);
}

}  // namespace

extern "C" {

int xb_rsvd_dense(xb_ctx* c, int dtype, int64_t m, int64_t n, const void* A, int64_t lda,
                  const void* omega, uint64_t seed, int k, int p, int q, void* U, int64_t ldu,
                  double* s, void* V, int64_t ldv, int32_t* deficient, int* ndeficient,
                  double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    const bool f32 = check_dtype(dtype);
    const size_t es = f32 ? 4 : 8;
    check_dims(m, n, k, p, q);
    XB_REQUIRE(A && U && s && V, XB_EVALUE, "null buffer");
    XB_REQUIRE(lda >= n && ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    ContiguousSource src(A, lda, n, es);
    rsvd_from_host(c, f32, m, n, src, 0, g_force_stream_rows >= 0, g_force_stream_rows, omega,
                   seed, k, p, q, U, ldu, s, V, ldv, deficient, ndeficient, stage_seconds);
  });
}

int xb_rsvd_dense_tiles(xb_ctx* c, int dtype, int64_t m, int64_t n, const int64_t* row_cuts,
                        int ntr, const int64_t* col_cuts, int ntc, xb_tile_fetch_fn fetch,
                        xb_tile_release_fn release, void* user, int force_stream, uint64_t seed,
                        int k, int p, int q, void* U, int64_t ldu, double* s, void* V,
                        int64_t ldv, int32_t* deficient, int* ndeficient,
                        double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    const bool f32 = check_dtype(dtype);
    check_dims(m, n, k, p, q);
    XB_REQUIRE(U && s && V && fetch && row_cuts && col_cuts && ntr >= 1 && ntc >= 1, XB_EVALUE,
               "null argument");
    XB_REQUIRE(ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    XB_REQUIRE(row_cuts[0] == 0 && row_cuts[ntr] == m && col_cuts[0] == 0 && col_cuts[ntc] == n,
               XB_ESHAPE, "tile cuts must span the matrix");
    int64_t band = 0;
    for (int i = 0; i < ntr; ++i) {
      XB_REQUIRE(row_cuts[i + 1] > row_cuts[i], XB_ESHAPE, "row cuts must increase");
      band = std::max(band, row_cuts[i + 1] - row_cuts[i]);
    }
    for (int j = 0; j < ntc; ++j)
      XB_REQUIRE(col_cuts[j + 1] > col_cuts[j], XB_ESHAPE, "column cuts must increase");
    TileSource src(row_cuts, ntr, col_cuts, ntc, fetch, release, user, f32 ? 4 : 8);
    rsvd_from_host(c, f32, m, n, src, band, force_stream != 0, 0, nullptr, seed, k, p, q, U, ldu,
                   s, V, ldv, deficient, ndeficient, stage_seconds);
  });
}

int xb_rsvd_dense_streamed(xb_ctx* c, int dtype, int64_t m, int64_t n, const void* A,
                           int64_t lda, uint64_t seed, int k, int p, int q, int64_t tile_rows,
                           void* U, int64_t ldu, double* s, void* V, int64_t ldv,
                           int32_t* deficient, int* ndeficient, double* stage_seconds) {
  if (tile_rows < 0) {
    g_last_error = "tile_rows must be >= 0";
    return XB_EVALUE;
  }
  g_force_stream_rows = tile_rows;
  const int rc = xb_rsvd_dense(c, dtype, m, n, A, lda, nullptr, seed, k, p, q, U, ldu, s, V, ldv,
                               deficient, ndeficient, stage_seconds);
  g_force_stream_rows = -1;
  return rc;
}

}  // extern "C"

namespace {

// Device CSR of A plus the once-built CSR of A^T (ingest, "Text Parsing").
AOp sparse_op(xb_ctx* c, int64_t m, int64_t n, int64_t nnz, const int64_t* d_rowptr,
              const int32_t* d_col, const double* d_val) {
  AOp op;
  op.sparse = true;
  op.csr = Csr{m, n, nnz, d_rowptr, d_col, d_val};
  auto* tptr = static_cast<int64_t*>(c->buf("t_ptr", (size_t)(n + 1) * 8));
  auto* trow = static_cast<int32_t*>(c->buf("t_row", (size_t)std::max<int64_t>(nnz, 1) * 4));
  double* tval = c->dbuf("t_val", (size_t)std::max<int64_t>(nnz, 1));
  auto* scr = static_cast<unsigned long long*>(c->buf("t_scr", (size_t)(n + 1) * 8));
  launch_csr_transpose(op.csr, tptr, trow, tval, scr, c->st);
  op.csrt = Csr{n, m, nnz, tptr, trow, tval};
  return op;
}

// Host COO -> device CSR (+ A^T). Returns the operator; timing into stage 0.
AOp sparse_from_host_coo(xb_ctx* c, int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                         const int64_t* cols, const double* vals) {
  XB_REQUIRE(m >= 1 && n >= 1 && nnz >= 0, XB_ESHAPE, "bad sparse shape");
  XB_REQUIRE(n < (int64_t)1 << 31 && m < (int64_t)1 << 31, XB_EUNSUPPORTED,
             "sparse dimensions must fit int32 column indices");
  const size_t nz = (size_t)std::max<int64_t>(nnz, 1);
  auto* drows = static_cast<int64_t*>(c->buf("coo_r", nz * 8));
  auto* dcols = static_cast<int64_t*>(c->buf("coo_c", nz * 8));
  double* dval = c->dbuf("csr_v", nz);
  auto* rowptr = static_cast<int64_t*>(c->buf("csr_p", (size_t)(m + 1) * 8));
  auto* col32 = static_cast<int32_t*>(c->buf("csr_c", nz * 4));
  if (nnz > 0) {
    // pageable arrays of >= 32 MB go through the staging ring (a pageable
    // cudaMemcpy runs at ~10 GB/s: 46 ms for cfg3's 480 MB)
    auto h2d = [&](void* d, const void* h) {
      const size_t bytes = (size_t)nnz * 8;
      if (bytes < ((size_t)32 << 20) || is_pinned(h)) {
        XB_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->st));
        return;
      }
      if (!c->stager)
        c->stager = new HostStager(stage_threads(), stage_slots(), stage_slot_bytes(),
                                   stage_piece_bytes());
      // rows of one staging piece each: the ring splits them over its slots
      const size_t w = c->stager->kPiece;
      const int64_t full = (int64_t)(bytes / w);
      if (full > 0)
        c->stager->copy(static_cast<char*>(d), w, static_cast<const char*>(h), w, w, full, c->st);
      if (bytes % w)
        c->stager->copy(static_cast<char*>(d) + (size_t)full * w, bytes % w,
                        static_cast<const char*>(h) + (size_t)full * w, bytes % w, bytes % w, 1,
                        c->st);
    };
    h2d(drows, rows);
    h2d(dcols, cols);
    h2d(dval, vals);
  }
  launch_coo_to_csr(drows, dcols, nnz, m, rowptr, col32, c->st);
  return sparse_op(c, m, n, nnz, rowptr, col32, dval);
}

}  // namespace

extern "C" {

int xb_comm_unique_id(unsigned char* out128) {
  return guarded([&] {
    XB_REQUIRE(out128, XB_EVALUE, "null buffer");
    nccl_unique_id(out128);
  });
}

int xb_comm_init(xb_ctx* c, const unsigned char* id128, int world, int rank) {
  return guarded([&] {
    XB_REQUIRE(c && id128, XB_EVALUE, "null argument");
    XB_REQUIRE(world >= 1 && rank >= 0 && rank < world, XB_EVALUE, "bad rank/world");
    LaunchScope ls(c);
    delete c->comm;
    c->comm = nullptr;
    c->comm = nccl_comm_create(id128, world, rank);
    c->world = world;
    c->rank = rank;
  });
}

int xb_comm_init_host(xb_ctx* c, int world, int rank, xb_host_collective_fn fn, void* user) {
  return guarded([&] {
    XB_REQUIRE(c && fn, XB_EVALUE, "null argument");
    XB_REQUIRE(world >= 1 && rank >= 0 && rank < world, XB_EVALUE, "bad rank/world");
    LaunchScope ls(c);
    delete c->comm;
    c->comm = nullptr;
    c->comm = host_comm_create(world, rank, fn, user);
    c->world = world;
    c->rank = rank;
  });
}

int xb_rsvd_dense_sharded_dev(xb_ctx* c, int dtype, int64_t m_global, int64_t n, int64_t m_local,
                              const void* dA, int64_t lda, uint64_t seed, int k, int p, int q,
                              void* dU, int64_t ldu, double* d_s, void* dV, int64_t ldv,
                              int32_t* deficient, int* ndeficient, double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    XB_REQUIRE(c->comm, XB_EVALUE, "xb_comm_init has not been called on this context");
    LaunchScope ls(c);
    after_caller_stream(c);
    const bool f32 = check_dtype(dtype);
    XB_REQUIRE(m_local >= 1 && m_local <= m_global, XB_ESHAPE, "bad local row count");
    XB_REQUIRE(lda >= n && ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    AOp op;
    op.dense = AView{dA, lda, f32};
    op.comm = c->comm;
    op.m_global = m_global;
    double* Ud = f32 ? c->dbuf("Ud", (size_t)m_local * k) : static_cast<double*>(dU);
    double* Vd = f32 ? c->dbuf("Vd", (size_t)n * k) : static_cast<double*>(dV);
    RsvdOut out{Ud, f32 ? k : ldu, d_s, Vd, f32 ? k : ldv};
    rsvd_impl(c, op, m_local, n, nullptr, k + p, seed, k, p, q, out, deficient, ndeficient,
              stage_seconds, IngestPlan{});
    if (f32) {
      launch_copy2d_cast<double, float>(Ud, m_local, k, k, static_cast<float*>(dU), ldu, c->st);
      launch_copy2d_cast<double, float>(Vd, n, k, k, static_cast<float*>(dV), ldv, c->st);
      XB_CUDA(cudaStreamSynchronize(c->st));
    }
  });
}

int xb_rsvd_dense_colsharded_dev(xb_ctx* c, int dtype, int64_t m, int64_t n_global,
                                 int64_t n_local, int64_t col0, const void* dA, int64_t lda,
                                 uint64_t seed, int k, int p, int q, void* dU, int64_t ldu,
                                 double* d_s, void* dV, int64_t ldv, int32_t* deficient,
                                 int* ndeficient, double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    XB_REQUIRE(c->comm, XB_EVALUE, "xb_comm_init has not been called on this context");
    LaunchScope ls(c);
    after_caller_stream(c);
    const bool f32 = check_dtype(dtype);
    XB_REQUIRE(n_local >= 1 && col0 >= 0 && col0 + n_local <= n_global, XB_ESHAPE,
               "bad local column block");
    XB_REQUIRE(lda >= n_local && ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    AOp op;
    op.dense = AView{dA, lda, f32};
    op.comm = c->comm;
    op.col_shard = true;
    op.n_global = n_global;
    op.col0 = col0;
    double* Ud = f32 ? c->dbuf("Ud", (size_t)m * k) : static_cast<double*>(dU);
    double* Vd = f32 ? c->dbuf("Vd", (size_t)n_local * k) : static_cast<double*>(dV);
    RsvdOut out{Ud, f32 ? k : ldu, d_s, Vd, f32 ? k : ldv};
    rsvd_impl(c, op, m, n_local, nullptr, k + p, seed, k, p, q, out, deficient, ndeficient,
              stage_seconds, IngestPlan{});
    if (f32) {
      launch_copy2d_cast<double, float>(Ud, m, k, k, static_cast<float*>(dU), ldu, c->st);
      launch_copy2d_cast<double, float>(Vd, n_local, k, k, static_cast<float*>(dV), ldv, c->st);
      XB_CUDA(cudaStreamSynchronize(c->st));
    }
  });
}

int xb_rsvd_csr_dev(xb_ctx* c, int64_t m, int64_t n, int64_t nnz, const int64_t* d_rowptr,
                    const int32_t* d_col, const double* d_val, const double* d_omega,
                    uint64_t seed, int k, int p, int q, double* dU, int64_t ldu, double* d_s,
                    double* dV, int64_t ldv, int32_t* deficient, int* ndeficient,
                    double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    after_caller_stream(c);
    check_dims(m, n, k, p, q);
    XB_REQUIRE(ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    AOp op = sparse_op(c, m, n, nnz, d_rowptr, d_col, d_val);
    RsvdOut out{dU, ldu, d_s, dV, ldv};
    rsvd_impl(c, op, m, n, d_omega, k + p, seed, k, p, q, out, deficient, ndeficient,
              stage_seconds, IngestPlan{});
  });
}

int xb_rsvd_csr_sharded_dev(xb_ctx* c, int64_t m_global, int64_t n, int64_t m_local,
                            int64_t nnz, const int64_t* d_rowptr, const int32_t* d_col,
                            const double* d_val, uint64_t seed, int k, int p, int q, double* dU,
                            int64_t ldu, double* d_s, double* dV, int64_t ldv,
                            int32_t* deficient, int* ndeficient, double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    XB_REQUIRE(c->comm, XB_EVALUE, "xb_comm_init has not been called on this context");
    LaunchScope ls(c);
    after_caller_stream(c);
    XB_REQUIRE(m_local >= 1 && m_local <= m_global, XB_ESHAPE, "bad local row count");
    XB_REQUIRE(ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    // this rank's rows of A as CSR (rowptr relative to its first row); the
    // A^T partials (n x l) are summed over ranks after every TN product
    AOp op = sparse_op(c, m_local, n, nnz, d_rowptr, d_col, d_val);
    op.comm = c->comm;
    op.m_global = m_global;
    RsvdOut out{dU, ldu, d_s, dV, ldv};
    rsvd_impl(c, op, m_local, n, nullptr, k + p, seed, k, p, q, out, deficient, ndeficient,
              stage_seconds, IngestPlan{});
  });
}

int xb_coo_sorted(const int64_t* rows, const int64_t* cols, int64_t nnz, int* sorted) {
  return guarded([&] {
    XB_REQUIRE(sorted && (nnz == 0 || (rows && cols)), XB_EVALUE, "null argument");
    // strictly increasing (row, col): the SparseBlock invariant (core.py:245-284),
    // checked on host threads (numpy's vectorised test of 2e7 entries took 70 ms
    // of a 210 ms cfg3 call)
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(stage_threads(), nnz >> 20));
    std::vector<int> bad(nt, 0);
    auto scan = [&](int t) {
      const int64_t lo = std::max<int64_t>(1, nnz * t / nt), hi = nnz * (t + 1) / nt;
      int b = 0;
      for (int64_t i = lo; i < hi; ++i)
        b |= !(rows[i] > rows[i - 1] || (rows[i] == rows[i - 1] && cols[i] > cols[i - 1]));
      bad[t] = b;
    };
    std::vector<std::thread> ts;
    for (int t = 1; t < nt; ++t) ts.emplace_back(scan, t);
    scan(0);
    for (auto& th : ts) th.join();
    int any = 0;
    for (int b : bad) any |= b;
    *sorted = !any;
  });
}

int xb_rsvd_coo(xb_ctx* c, int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                const int64_t* cols, const double* vals, const double* omega, uint64_t seed,
                int k, int p, int q, double* U, int64_t ldu, double* s, double* V, int64_t ldv,
                int32_t* deficient, int* ndeficient, double* stage_seconds) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    check_dims(m, n, k, p, q);
    XB_REQUIRE(U && s && V && (nnz == 0 || (rows && cols && vals)), XB_EVALUE, "null buffer");
    XB_REQUIRE(ldu >= k && ldv >= k, XB_EVALUE, "leading dimension too small");
    const int l = k + p;
    OutputPretouch touch(U, (size_t)ldu * 8, (size_t)k * 8, m, V, (size_t)ldv * 8, (size_t)k * 8, n);
    cudaEvent_t e0, e1;
    XB_CUDA(cudaEventCreate(&e0));
    XB_CUDA(cudaEventCreate(&e1));
    XB_CUDA(cudaEventRecord(e0, c->st));
    AOp op = sparse_from_host_coo(c, m, n, nnz, rows, cols, vals);
    XB_CUDA(cudaEventRecord(e1, c->st));
    double* dU = c->dbuf("U", (size_t)m * k);
    double* dV = c->dbuf("V", (size_t)n * k);
    double* ds = c->dbuf("s", (size_t)k);
    double* dO = nullptr;
    if (omega) {
      dO = c->dbuf("omega_in", (size_t)n * l);
      XB_CUDA(cudaMemcpyAsync(dO, omega, (size_t)n * l * 8, cudaMemcpyHostToDevice, c->st));
    }
    RsvdOut out{dU, k, ds, dV, k};
    rsvd_impl(c, op, m, n, dO, l, seed, k, p, q, out, deficient, ndeficient, stage_seconds,
              IngestPlan{});
    XB_CUDA(cudaMemcpyAsync(s, ds, k * 8, cudaMemcpyDeviceToHost, c->st));
    touch.join();
    d2h_rows(c, U, ldu * 8, dU, k * 8, k * 8, m);
    d2h_rows(c, V, ldv * 8, dV, k * 8, k * 8, n);
    XB_CUDA(cudaStreamSynchronize(c->st));
    float ms = 0.f;
    XB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (stage_seconds) stage_seconds[kParse] += ms * 1e-3;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

int xb_spmm_coo(xb_ctx* c, int64_t m, int64_t n, int64_t nnz, const int64_t* rows,
                const int64_t* cols, const double* vals, int trans, const double* X, int64_t l,
                double* Y) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    XB_REQUIRE(l >= 1 && l <= 576, XB_EUNSUPPORTED, "spmm: 1 <= l <= 576");
    AOp op = sparse_from_host_coo(c, m, n, nnz, rows, cols, vals);
    const Csr& s = trans ? op.csrt : op.csr;
    double* dX = c->dbuf("spX", (size_t)s.cols * l);
    double* dY = c->dbuf("spY", (size_t)s.rows * l);
    XB_CUDA(cudaMemcpyAsync(dX, X, (size_t)s.cols * l * 8, cudaMemcpyHostToDevice, c->st));
    launch_spmm(s, dX, l, dY, l, (int)l, c->st);
    XB_CUDA(cudaMemcpyAsync(Y, dY, (size_t)s.rows * l * 8, cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
  });
}

int xb_gaussian(xb_ctx* c, int dtype, uint64_t seed, int64_t row0, int64_t rows, int64_t cols,
                void* out, int64_t ld) {
  return guarded([&] {
    XB_REQUIRE(c && out, XB_EVALUE, "null argument");
    LaunchScope ls(c);
    XB_REQUIRE(rows >= 0 && cols >= 1 && ld >= cols && row0 >= 0, XB_EVALUE, "bad shape");
    if (rows == 0) return;
    const size_t es = dtype == XB_F64 ? 8 : 4;
    XB_REQUIRE(dtype == XB_F64 || dtype == XB_F32, XB_EVALUE, "unknown dtype");
    void* d = c->buf("gauss_out", (size_t)rows * cols * es);
    if (dtype == XB_F64)
      launch_gaussian<double>(seed, row0, rows, cols, static_cast<double*>(d), cols, cols, c->st);
    else
      launch_gaussian<float>(seed, row0, rows, cols, static_cast<float*>(d), cols, cols, c->st);
    XB_CUDA(cudaMemcpy2DAsync(out, ld * es, d, cols * es, cols * es, rows, cudaMemcpyDeviceToHost,
                              c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
  });
}

int xb_uniform_bits(xb_ctx* c, uint64_t seed, int64_t row0, int64_t rows, int64_t cols,
                    uint64_t* out) {
  return guarded([&] {
    XB_REQUIRE(c && out, XB_EVALUE, "null argument");
    LaunchScope ls(c);
    XB_REQUIRE(rows >= 0 && cols >= 1 && row0 >= 0, XB_EVALUE, "bad shape");
    if (rows == 0) return;
    const int64_t count = 2 * ((cols + 1) / 2);
    auto* d = static_cast<uint64_t*>(c->buf("bits_out", (size_t)rows * count * 8));
    launch_uniform_bits(seed, row0, rows, cols, d, c->st);
    XB_CUDA(cudaMemcpyAsync(out, d, (size_t)rows * count * 8, cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
  });
}

int xb_gemm_dev(xb_ctx* c, int dtype, int trans_a, int64_t m, int64_t n, int64_t kdim,
                const void* dA, int64_t lda, const void* dB, int64_t ldb, void* dC, int64_t ldc) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    after_caller_stream(c);
    const bool f32 = check_dtype(dtype);
    XB_REQUIRE(m >= 0 && n >= 0 && kdim >= 0, XB_ESHAPE, "negative dimension");
    XB_REQUIRE(ldc >= n && ldb >= n && lda >= (trans_a ? m : kdim), XB_EVALUE,
               "leading dimension too small");
    if (m == 0 || n == 0) return;
    gemm_any(c, f32, trans_a != 0, m, n, kdim, dA, lda, dB, ldb, dC, ldc);
    XB_CUDA(cudaStreamSynchronize(c->st));
  });
}

int xb_gemm(xb_ctx* c, int dtype, int trans_a, int64_t m, int64_t n, int64_t kdim, const void* A,
            int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    const bool f32 = check_dtype(dtype);
    const size_t es = f32 ? 4 : 8;
    XB_REQUIRE(m >= 0 && n >= 0 && kdim >= 0, XB_ESHAPE, "negative dimension");
    XB_REQUIRE(ldc >= n && ldb >= n && lda >= (trans_a ? m : kdim), XB_EVALUE,
               "leading dimension too small");
    if (m == 0 || n == 0) return;
    const int64_t arows = trans_a ? kdim : m, acols = trans_a ? m : kdim;
    void* dA = c->buf("gA", (size_t)std::max<int64_t>(1, arows * acols) * es);
    void* dB = c->buf("gB", (size_t)std::max<int64_t>(1, kdim * n) * es);
    void* dC = c->buf("gC", (size_t)m * n * es);
    if (arows * acols > 0)
      XB_CUDA(cudaMemcpy2DAsync(dA, acols * es, A, lda * es, acols * es, arows,
                                cudaMemcpyHostToDevice, c->st));
    if (kdim * n > 0)
      XB_CUDA(cudaMemcpy2DAsync(dB, n * es, B, ldb * es, n * es, kdim, cudaMemcpyHostToDevice,
                                c->st));
    gemm_any(c, f32, trans_a != 0, m, n, kdim, dA, acols, dB, n, dC, n);
    XB_CUDA(cudaMemcpy2DAsync(C, ldc * es, dC, n * es, n * es, m, cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
  });
}

int xb_thin_qr(xb_ctx* c, int dtype, int64_t m, int64_t r, const void* Y, int64_t ldy, void* Q,
               int64_t ldq, double* R, int32_t* deficient, int* ndeficient) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    const bool f32 = check_dtype(dtype);
    XB_REQUIRE(r >= 1 && m >= r, XB_ESHAPE,
               "thin QR needs rows >= cols >= 1, got " + std::to_string(m) + "x" +
                   std::to_string(r));
    XB_REQUIRE(ldy >= r && ldq >= r, XB_EVALUE, "leading dimension too small");
    const int l = (int)r, lp = (int)round_up(r, 8);
    double* dY = c->dbuf("qrY", (size_t)m * lp);
    double* dT = c->dbuf("qrT", (size_t)m * lp);
    double* dQ = c->dbuf("qrQ", (size_t)m * lp);
    double* dR = c->dbuf("qrR", (size_t)lp * lp);
    int* defc = c->ibuf("qrdef", (size_t)lp + 4);
    c->dbuf("tsqr_work", tsqr_work_doubles(m, l));
    XB_CUDA(cudaMemsetAsync(dY, 0, (size_t)m * lp * 8, c->st));
    // the reference factors in f64 whatever the storage precision (kernels.py:308-316)
    if (f32) {
      float* y32 = static_cast<float*>(c->buf("qrY32", (size_t)m * r * 4));
      XB_CUDA(cudaMemcpy2DAsync(y32, r * 4, Y, ldy * 4, r * 4, m, cudaMemcpyHostToDevice, c->st));
      launch_copy2d_cast<float, double>(y32, m, r, r, dY, lp, c->st);
    } else {
      XB_CUDA(cudaMemcpy2DAsync(dY, lp * 8, Y, ldy * 8, r * 8, m, cudaMemcpyHostToDevice, c->st));
    }
    Small s = small_bufs(c, l);
    cholqr2(c, s, dY, m, dT, dQ, dR);
    // compute-dtype eps for the deficiency threshold (kernels.py:328)
    launch_deficient(dR, lp, l, f32 ? (double)FLT_EPSILON : DBL_EPSILON, defc, defc + 1, c->st);
    std::vector<int> hdef(lp + 1, 0);
    if (f32) {
      float* q32 = static_cast<float*>(c->buf("qrQ32", (size_t)m * r * 4));
      launch_copy2d_cast<double, float>(dQ, m, r, lp, q32, r, c->st);
      XB_CUDA(cudaMemcpy2DAsync(Q, ldq * 4, q32, r * 4, r * 4, m, cudaMemcpyDeviceToHost, c->st));
    } else {
      XB_CUDA(cudaMemcpy2DAsync(Q, ldq * 8, dQ, lp * 8, r * 8, m, cudaMemcpyDeviceToHost, c->st));
    }
    if (R)
      XB_CUDA(cudaMemcpy2DAsync(R, r * 8, dR, lp * 8, r * 8, r, cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaMemcpyAsync(hdef.data(), defc, (lp + 1) * sizeof(int), cudaMemcpyDeviceToHost,
                            c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
    if (ndeficient) *ndeficient = hdef[0];
    if (deficient)
      for (int i = 0; i < hdef[0] && i < l; ++i) deficient[i] = hdef[1 + i];
  });
}

int xb_tsqr_dev(xb_ctx* c, int64_t m, int64_t r, const double* dY, int64_t ldy, double* dQ,
                int64_t ldq, double* dR, int64_t ldr, int32_t* deficient, int* ndeficient,
                double* seconds) {
  return guarded([&] {
    XB_REQUIRE(c && dY && dQ && dR, XB_EVALUE, "null argument");
    LaunchScope ls(c);
    after_caller_stream(c);
    XB_REQUIRE(r >= 1 && m >= r, XB_ESHAPE,
               "TSQR needs rows >= cols >= 1, got " + std::to_string(m) + "x" + std::to_string(r));
    XB_REQUIRE(ldy >= r && ldq >= r && ldr >= r, XB_EVALUE, "leading dimension too small");
    const int l = (int)r;
    double* w = c->dbuf("tsqr_work", tsqr_work_doubles(m, l));
    int* defc = c->ibuf("qrdef", (size_t)l + 4);
    cudaEvent_t e0, e1;
    XB_CUDA(cudaEventCreate(&e0));
    XB_CUDA(cudaEventCreate(&e1));
    XB_CUDA(cudaEventRecord(e0, c->st));
    launch_tsqr(dY, ldy, m, l, l, dQ, ldq, dR, ldr, w, nullptr, c->st);
    XB_CUDA(cudaEventRecord(e1, c->st));
    launch_deficient(dR, ldr, l, DBL_EPSILON, defc, defc + 1, c->st);
    std::vector<int> hdef(l + 1, 0);
    XB_CUDA(cudaMemcpyAsync(hdef.data(), defc, (l + 1) * sizeof(int), cudaMemcpyDeviceToHost,
                            c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
    float ms = 0.f;
    XB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (seconds) *seconds = ms * 1e-3;
    if (ndeficient) *ndeficient = hdef[0];
    if (deficient)
      for (int i = 0; i < hdef[0] && i < l; ++i) deficient[i] = hdef[1 + i];
  });
}

int xb_svd_small(xb_ctx* c, int64_t r, int64_t n, const double* B, int64_t ldb, double* U,
                 double* s, double* V) {
  return guarded([&] {
    XB_REQUIRE(c, XB_EVALUE, "null context");
    LaunchScope ls(c);
    XB_REQUIRE(r >= 1 && n >= 1, XB_ESHAPE, "svd_small expects a non-empty matrix");
    XB_REQUIRE(r <= n, XB_ESHAPE,
               "svd_small expects r <= n, got " + std::to_string(r) + "x" + std::to_string(n));
    XB_REQUIRE(ldb >= n, XB_EVALUE, "leading dimension too small");
    const int l = (int)r, lp = (int)round_up(r, 8);
    double* dB = c->dbuf("svB", (size_t)r * n);
    double* dBt = c->dbuf("svBt", (size_t)n * lp);
    double* dT = c->dbuf("svT", (size_t)n * lp);
    double* dQ = c->dbuf("svQ", (size_t)n * lp);
    double* dR = c->dbuf("svR", (size_t)lp * lp);
    double* dUb = c->dbuf("svU", (size_t)lp * lp);
    double* dW = c->dbuf("svW", (size_t)lp * lp);
    double* ds = c->dbuf("svs", (size_t)lp);
    double* dV = c->dbuf("svV", (size_t)n * l);
    double* jw = c->dbuf("jw", jacobi_work_doubles(lp));
    int* jstat = c->ibuf("jstat", 4);
    c->dbuf("tsqr_work", tsqr_work_doubles(n, l));
    XB_CUDA(cudaMemcpy2DAsync(dB, n * 8, B, ldb * 8, n * 8, r, cudaMemcpyHostToDevice, c->st));
    XB_CUDA(cudaMemsetAsync(dBt, 0, (size_t)n * lp * 8, c->st));
    XB_CUDA(cudaMemsetAsync(dUb, 0, (size_t)lp * lp * 8, c->st));
    XB_CUDA(cudaMemsetAsync(dW, 0, (size_t)lp * lp * 8, c->st));
    launch_transpose(dB, r, n, n, dBt, lp, c->st);
    Small sm = small_bufs(c, l);
    cholqr2(c, sm, dBt, n, dT, dQ, dR);
    launch_jacobi_svd(dR, lp, l, l, dUb, lp, ds, dW, lp, jw, jstat, c->st);
    gemm(c, false, n, l, lp, dQ, lp, dW, lp, dV, l);
    int hstat = 0;
    XB_CUDA(cudaMemcpy2DAsync(U, r * 8, dUb, lp * 8, r * 8, r, cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaMemcpyAsync(s, ds, r * 8, cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaMemcpyAsync(V, dV, (size_t)n * r * 8, cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaMemcpyAsync(&hstat, jstat, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    XB_CUDA(cudaStreamSynchronize(c->st));
    XB_REQUIRE(hstat == 0, XB_ECONV, "bidiagonal SVD did not converge in 60 sweeps");
  });
}

}  // extern "C"

namespace xb {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace xb
