"""ctypes binding of the C ABI (include/xsvd_b200.h).

The library is REQUIRED: there is no CPU fallback anywhere in this package.
`load()` raises XsvdError when libxsvdb200.so is missing or no CUDA device is
usable, so a product call on a machine without the CUDA path fails loudly.
ctypes releases the GIL for the duration of every call.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import XsvdError, raise_for_status

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libxsvdb200.so")

XB_F32, XB_F64 = 1, 2
NUM_STAGES = 8
POWER_AUTO = -1  # XB_POWER_AUTO: q argument selecting power = "auto"
COLL_ALLREDUCE_SUM, COLL_ALLGATHER = 0, 1  # xb_host_collective_fn ops
HOST_COLLECTIVE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int64)
TILE_FETCH = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_int64))
TILE_RELEASE = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int64)

_lock = threading.Lock()
_lib = None
_ctxs: dict[int, "Context"] = {}

# (name, restype, argtypes) for every symbol include/xsvd_b200.h declares
_i64, _u64, _int, _vp, _dp = C.c_int64, C.c_uint64, C.c_int, C.c_void_p, C.POINTER(C.c_double)
_i32p, _intp = C.POINTER(C.c_int32), C.POINTER(C.c_int)
SIGNATURES = [
    ("xb_abi_version", _int, []),
    ("xb_build_flags", _int, []),
    ("xb_last_error", C.c_char_p, []),
    ("xb_create", _int, [_int, C.POINTER(_vp)]),
    ("xb_destroy", _int, [_vp]),
    ("xb_launch_count", _i64, [_vp]),
    ("xb_compute_stream", _vp, [_vp]),
    ("xb_profile_enable", _int, [_vp, _int]),
    ("xb_profile_read", _int, [_vp, _vp]),
    ("xb_profile_read_ext", _int, [_vp, _vp]),
    ("xb_fp64_peaks", _int, [_vp, _dp, _dp]),
    ("xb_tc_peaks", _int, [_vp, _dp, _dp]),
    ("xb_tc_peaks_data", _int, [_vp, _int, _dp, _dp]),
    ("xb_coo_sorted", _int, [_vp, _vp, C.c_int64, C.POINTER(C.c_int)]),
    ("xb_set_power_auto", _int, [_vp, _int, C.c_double]),
    ("xb_last_power", _int, [_vp, _intp, _vp, _int, _intp]),
    ("xb_set_gram_path", _int, [_vp, _int]),
    ("xb_rsvd_dense", _int, [_vp, _int, _i64, _i64, _vp, _i64, _vp, _u64, _int, _int, _int,
                             _vp, _i64, _vp, _vp, _i64, _vp, _intp, _vp]),
    ("xb_rsvd_dense_dev", _int, [_vp, _int, _i64, _i64, _vp, _i64, _vp, _u64, _int, _int, _int,
                                 _vp, _i64, _vp, _vp, _i64, _vp, _intp, _vp]),
    ("xb_rsvd_dense_tiles", _int, [_vp, _int, _i64, _i64, _vp, _int, _vp, _int, _vp, _vp, _vp,
                                   _int, _u64, _int, _int, _int, _vp, _i64, _vp, _vp, _i64, _vp,
                                   _intp, _vp]),
    ("xb_rsvd_dense_streamed", _int, [_vp, _int, _i64, _i64, _vp, _i64, _u64, _int, _int, _int,
                                      _i64, _vp, _i64, _vp, _vp, _i64, _vp, _intp, _vp]),
    ("xb_comm_unique_id", _int, [_vp]),
    ("xb_comm_init", _int, [_vp, _vp, _int, _int]),
    ("xb_rsvd_dense_sharded_dev", _int, [_vp, _int, _i64, _i64, _i64, _vp, _i64, _u64, _int, _int,
                                         _int, _vp, _i64, _vp, _vp, _i64, _vp, _intp, _vp]),
    ("xb_rsvd_dense_colsharded_dev", _int, [_vp, _int, _i64, _i64, _i64, _i64, _vp, _i64, _u64,
                                            _int, _int, _int, _vp, _i64, _vp, _vp, _i64, _vp,
                                            _intp, _vp]),
    ("xb_rsvd_coo", _int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _u64, _int, _int, _int,
                           _vp, _i64, _vp, _vp, _i64, _vp, _intp, _vp]),
    ("xb_rsvd_csr_sharded_dev", _int, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _u64, _int,
                                       _int, _int, _vp, _i64, _vp, _vp, _i64, _vp, _intp, _vp]),
    ("xb_rsvd_csr_dev", _int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _u64, _int, _int, _int,
                               _vp, _i64, _vp, _vp, _i64, _vp, _intp, _vp]),
    ("xb_spmm_coo", _int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _int, _vp, _i64, _vp]),
    ("xb_gaussian", _int, [_vp, _int, _u64, _i64, _i64, _i64, _vp, _i64]),
    ("xb_uniform_bits", _int, [_vp, _u64, _i64, _i64, _i64, _vp]),
    ("xb_gemm", _int, [_vp, _int, _int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    ("xb_gemm_dev", _int, [_vp, _int, _int, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    ("xb_thin_qr", _int, [_vp, _int, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _intp]),
    ("xb_svd_small", _int, [_vp, _i64, _i64, _vp, _i64, _vp, _vp, _vp]),
    ("xb_tsqr_dev", _int, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _intp, _vp]),
    ("xb_comm_init_host", _int, [_vp, _int, _int, _vp, _vp]),
    ("xb_mm_info", _int, [C.c_char_p, _vp, _vp, _vp, _intp, _intp, _vp]),
    ("xb_mm_read", _int, [C.c_char_p, _int, _i64, _vp, _vp]),
    ("xb_coo_free", None, [_vp]),
]


class XbCoo(C.Structure):
    """xb_coo (include/xsvd_b200.h)."""
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("r", C.POINTER(C.c_int64)), ("c", C.POINTER(C.c_int64)),
                ("v", C.POINTER(C.c_double)), ("field", C.c_int), ("symmetric", C.c_int)]


FIELDS = {0: "real", 1: "integer", 2: "pattern"}


def mm_info(path: str) -> dict:
    """Matrix Market header + size line (xb_mm_info; no device needed)."""
    lib = lib_handle()
    rows, cols, ent, line = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    field, sym = C.c_int(), C.c_int()
    st = lib.xb_mm_info(os.fsencode(path), C.byref(rows), C.byref(cols), C.byref(ent),
                        C.byref(field), C.byref(sym), C.byref(line))
    if st != 0:
        raise_for_status(st, lib.xb_last_error().decode(errors="replace"), line.value or None)
    return {"rows": rows.value, "cols": cols.value, "entries": ent.value,
            "field": FIELDS[field.value], "symmetric": bool(sym.value)}


def mm_read(path: str, threads: int = 0, chunk_lines: int = 0):
    """Parse a Matrix Market coordinate file natively (xb_mm_read): returns
    (rows, cols, r, c, v, info) with 0-based int64 triplets in the
    reference's order, duplicates not yet summed."""
    lib = lib_handle()
    coo = XbCoo()
    line = C.c_int64()
    st = lib.xb_mm_read(os.fsencode(path), int(threads), int(chunk_lines), C.byref(coo),
                        C.byref(line))
    if st != 0:
        raise_for_status(st, lib.xb_last_error().decode(errors="replace"), line.value or None)
    try:
        n = coo.nnz
        r = np.ctypeslib.as_array(coo.r, shape=(n,)).copy() if n else np.zeros(0, np.int64)
        c = np.ctypeslib.as_array(coo.c, shape=(n,)).copy() if n else np.zeros(0, np.int64)
        v = np.ctypeslib.as_array(coo.v, shape=(n,)).copy() if n else np.zeros(0)
    finally:
        lib.xb_coo_free(C.byref(coo))
    return coo.rows, coo.cols, r, c, v, {"field": FIELDS[coo.field],
                                         "symmetric": bool(coo.symmetric)}


def lib_handle():
    """dlopen the library and bind every symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise XsvdError(
                    f"CUDA library missing: {LIB_PATH} (run __graft_entry__.build()); "
                    "this package has no CPU fallback")
            lib = C.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def _check(status: int):
    if status != 0:
        msg = lib_handle().xb_last_error().decode(errors="replace")
        raise_for_status(status, msg)


_MADV_HUGEPAGE = 14
try:
    _libc = C.CDLL(None, use_errno=True)
    _libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
    _libc.madvise.restype = C.c_int
except (OSError, AttributeError):  # pragma: no cover - no libc madvise
    _libc = None


def _out(shape, dtype=np.float64) -> np.ndarray:
    """A fresh output array for the library to fill. Large ones ask for
    transparent huge pages first: the device -> host copy is the first touch
    of every page, and 4 KiB first-touch faults (serialised on the process's
    mmap lock) capped a 0.96 GB result at ~7 GB/s."""
    a = np.empty(shape, dtype=dtype)
    if _libc is not None and a.nbytes >= (8 << 20):
        page = 2 << 20
        lo = (a.ctypes.data + page - 1) & ~(page - 1)
        hi = (a.ctypes.data + a.nbytes) & ~(page - 1)
        if hi > lo:
            _libc.madvise(C.c_void_p(lo), C.c_size_t(hi - lo), _MADV_HUGEPAGE)
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def dtype_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return XB_F64
    if dt == np.float32:
        return XB_F32
    raise XsvdError(f"unsupported dtype {dt}")


class Context:
    """One device's library context (streams + cached workspaces)."""

    def __init__(self, device: int):
        self.lib = lib_handle()
        self.device = device
        h = C.c_void_p()
        _check(self.lib.xb_create(device, C.byref(h)))
        self.h = h

    @property
    def launches(self) -> int:
        return int(self.lib.xb_launch_count(self.h))

    @property
    def stream_ptr(self) -> int:
        return int(self.lib.xb_compute_stream(self.h) or 0)

    def profile(self, on: bool):
        _check(self.lib.xb_profile_enable(self.h, int(on)))

    def profile_read(self) -> dict:
        out = np.zeros(6)
        _check(self.lib.xb_profile_read_ext(self.h, _ptr(out)))
        kinds = {0: "dmma", 1: "tf32x3", 2: "ozaki_i8", 3: "spmm", 4: "ozaki_f32_i8"}
        return {"seconds": out[0], "launches": int(out[1]), "flops": out[2], "bytes": out[3],
                "pipe_ops": out[4], "kind": kinds.get(int(out[5]))}

    def fp64_peaks(self):
        a, b = C.c_double(), C.c_double()
        _check(self.lib.xb_fp64_peaks(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def tc_peaks(self):
        """Measured dense tcgen05 rates: (int8 TOP/s, bf16 TFLOP/s)."""
        a, b = C.c_double(), C.c_double()
        _check(self.lib.xb_tc_peaks(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def tc_peaks_data(self, random_data: bool = True):
        """The same with random operand bytes (the power-limited rate on real data)."""
        a, b = C.c_double(), C.c_double()
        _check(self.lib.xb_tc_peaks_data(self.h, int(random_data), C.byref(a), C.byref(b)))
        return a.value, b.value

    # -- power selection ------------------------------------------------------
    def set_power_auto(self, q_max: int = 5, tau: float = 1e-6):
        """Stopping-rule parameters for calls made with q = POWER_AUTO."""
        _check(self.lib.xb_set_power_auto(self.h, int(q_max), float(tau)))

    def set_gram_path(self, on: bool):
        """RsvdConfig.gram_path for the following factorisations."""
        _check(self.lib.xb_set_gram_path(self.h, int(bool(on))))

    def last_power(self):
        """(chosen q, nu sequence) of the last factorisation."""
        q, cnt = C.c_int(0), C.c_int(0)
        nus = np.zeros(64)
        _check(self.lib.xb_last_power(self.h, C.byref(q), _ptr(nus), len(nus), C.byref(cnt)))
        return q.value, [float(x) for x in nus[: min(cnt.value, len(nus))]]

    # -- full factorisation ---------------------------------------------------
    def rsvd_dense(self, a: np.ndarray, k: int, p: int, q: int, seed: int, omega=None):
        """Host buffers in, host factors out (xb_rsvd_dense)."""
        a = np.asarray(a)
        if a.ndim != 2:
            raise XsvdError("A must be 2-d")
        if a.strides[1] != a.itemsize:
            a = np.ascontiguousarray(a)
        m, n = a.shape
        lda = a.strides[0] // a.itemsize
        dt = a.dtype
        l = k + p
        u = _out((m, k), dt)
        v = _out((n, k), dt)
        s = np.empty(k, dtype=np.float64)
        deficient = np.zeros(max(l, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES, dtype=np.float64)
        om = None
        if omega is not None:
            om = np.ascontiguousarray(omega, dtype=dt)
            if om.shape != (n, l):
                raise XsvdError(f"omega must be {(n, l)}, got {om.shape}")
        _check(self.lib.xb_rsvd_dense(
            self.h, dtype_code(dt), m, n, _ptr(a), lda, _ptr(om) if om is not None else None,
            int(seed) & (2**64 - 1), k, p, q, _ptr(u), k, _ptr(s), _ptr(v), k, _ptr(deficient),
            C.byref(ndef), _ptr(stages)))
        return u, s, v, tuple(int(x) for x in deficient[: ndef.value]), stages

    def rsvd_dense_tiles(self, shape, row_cuts, col_cuts, get_tile, dtype, k: int, p: int,
                         q: int, seed: int, release=None, force_stream: bool = False):
        """Dense A as a tile grid (xb_rsvd_dense_tiles): get_tile(ti, tj) ->
        2-d array of the tile (any row stride, unit column stride), held
        until the library releases it (then release(ti, tj), if given).
        A is never assembled in host memory."""
        m, n = shape
        dt = np.dtype(dtype)
        held = {}
        errors = []

        def fetch(user, ti, tj, ld_out):
            try:
                t = np.asarray(get_tile(int(ti), int(tj)))
                if t.dtype != dt or t.strides[1] != dt.itemsize:
                    t = np.ascontiguousarray(t, dtype=dt)
                held[(int(ti), int(tj))] = t
                ld_out[0] = t.strides[0] // dt.itemsize
                return t.ctypes.data
            except BaseException as e:  # noqa: BLE001 - reported as a null tile
                errors.append(e)
                return None

        def rel(user, ti, tj):
            held.pop((int(ti), int(tj)), None)
            if release is not None:
                release(int(ti), int(tj))

        fetch_cb, rel_cb = TILE_FETCH(fetch), TILE_RELEASE(rel)
        rc_ = np.ascontiguousarray(row_cuts, dtype=np.int64)
        cc_ = np.ascontiguousarray(col_cuts, dtype=np.int64)
        u = _out((m, k), dt)
        v = _out((n, k), dt)
        s = np.empty(k)
        deficient = np.zeros(max(k + p, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES)
        status = self.lib.xb_rsvd_dense_tiles(
            self.h, dtype_code(dt), m, n, _ptr(rc_), len(rc_) - 1, _ptr(cc_), len(cc_) - 1,
            fetch_cb, rel_cb, None, int(bool(force_stream)), int(seed) & (2**64 - 1), k, p, q,
            _ptr(u), k, _ptr(s), _ptr(v), k, _ptr(deficient), C.byref(ndef), _ptr(stages))
        if errors:
            raise errors[0]
        _check(status)
        return u, s, v, tuple(int(x) for x in deficient[: ndef.value]), stages

    def rsvd_dense_streamed(self, a: np.ndarray, k: int, p: int, q: int, seed: int,
                            tile_rows: int = 0):
        """Out-of-core factorisation: A stays in host memory and streams
        through HBM in row tiles (xb_rsvd_dense_streamed)."""
        a = np.asarray(a)
        if a.ndim != 2:
            raise XsvdError("A must be 2-d")
        if a.strides[1] != a.itemsize:
            a = np.ascontiguousarray(a)
        m, n = a.shape
        lda = a.strides[0] // a.itemsize
        dt = a.dtype
        u = _out((m, k), dt)
        v = _out((n, k), dt)
        s = np.empty(k)
        deficient = np.zeros(max(k + p, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES)
        _check(self.lib.xb_rsvd_dense_streamed(
            self.h, dtype_code(dt), m, n, _ptr(a), lda, int(seed) & (2**64 - 1), k, p, q,
            int(tile_rows), _ptr(u), k, _ptr(s), _ptr(v), k, _ptr(deficient), C.byref(ndef),
            _ptr(stages)))
        return u, s, v, tuple(int(x) for x in deficient[: ndef.value]), stages

    def rsvd_dense_dev(self, dtype, m, n, a_ptr, lda, k, p, q, seed, u_ptr, s_ptr, v_ptr,
                       omega_ptr=None):
        """Device pointers (e.g. torch tensors' data_ptr()) in and out."""
        deficient = np.zeros(max(k + p, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES, dtype=np.float64)
        _check(self.lib.xb_rsvd_dense_dev(
            self.h, dtype_code(dtype), m, n, C.c_void_p(a_ptr), lda,
            C.c_void_p(omega_ptr) if omega_ptr else None, int(seed) & (2**64 - 1), k, p, q,
            C.c_void_p(u_ptr), k, C.c_void_p(s_ptr), C.c_void_p(v_ptr), k, _ptr(deficient),
            C.byref(ndef), _ptr(stages)))
        return tuple(int(x) for x in deficient[: ndef.value]), stages

    # -- multi-GPU (row-sharded A) -----------------------------------------------------
    def comm_unique_id(self) -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(self.lib.xb_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, unique_id: bytes, world: int, rank: int):
        if len(unique_id) != 128:
            raise XsvdError("NCCL unique id must be 128 bytes")
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _check(self.lib.xb_comm_init(self.h, buf, world, rank))

    def rsvd_dense_sharded_dev(self, dtype, m_global, n, m_local, a_ptr, lda, k, p, q, seed,
                               u_ptr, s_ptr, v_ptr):
        deficient = np.zeros(max(k + p, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES)
        _check(self.lib.xb_rsvd_dense_sharded_dev(
            self.h, dtype_code(dtype), m_global, n, m_local, C.c_void_p(a_ptr), lda,
            int(seed) & (2**64 - 1), k, p, q, C.c_void_p(u_ptr), k, C.c_void_p(s_ptr),
            C.c_void_p(v_ptr), k, _ptr(deficient), C.byref(ndef), _ptr(stages)))
        return tuple(int(x) for x in deficient[: ndef.value]), stages

    def rsvd_dense_colsharded_dev(self, dtype, m, n_global, n_local, col0, a_ptr, lda, k, p, q,
                                  seed, u_ptr, s_ptr, v_ptr):
        deficient = np.zeros(max(k + p, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES)
        _check(self.lib.xb_rsvd_dense_colsharded_dev(
            self.h, dtype_code(dtype), m, n_global, n_local, col0, C.c_void_p(a_ptr), lda,
            int(seed) & (2**64 - 1), k, p, q, C.c_void_p(u_ptr), k, C.c_void_p(s_ptr),
            C.c_void_p(v_ptr), k, _ptr(deficient), C.byref(ndef), _ptr(stages)))
        return tuple(int(x) for x in deficient[: ndef.value]), stages

    # -- sparse A ----------------------------------------------------------------------
    @staticmethod
    def _coo(rows, cols, vals):
        """int64 (row, col)-sorted COO, the SparseBlock invariant (core.py:245-284)."""
        r = np.ascontiguousarray(rows, dtype=np.int64)
        c = np.ascontiguousarray(cols, dtype=np.int64)
        v = np.ascontiguousarray(vals, dtype=np.float64)
        ok = C.c_int(1)
        if len(r) > 1:
            _check(lib_handle().xb_coo_sorted(_ptr(r), _ptr(c), len(r), C.byref(ok)))
        if not ok.value:
            order = np.lexsort((c, r))
            r, c, v = r[order], c[order], v[order]
        return r, c, v

    def rsvd_coo(self, rows, cols, vals, shape, k, p, q, seed, omega=None):
        """Sparse A (COO host arrays) in, host factors out (xb_rsvd_coo)."""
        m, n = shape
        r, c, v = self._coo(rows, cols, vals)
        l = k + p
        u = _out((m, k))
        vv = _out((n, k))
        s = np.empty(k)
        deficient = np.zeros(max(l, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES)
        om = None
        if omega is not None:
            om = np.ascontiguousarray(omega, dtype=np.float64)
            if om.shape != (n, l):
                raise XsvdError(f"omega must be {(n, l)}, got {om.shape}")
        _check(self.lib.xb_rsvd_coo(
            self.h, m, n, len(v), _ptr(r), _ptr(c), _ptr(v), _ptr(om) if om is not None else None,
            int(seed) & (2**64 - 1), k, p, q, _ptr(u), k, _ptr(s), _ptr(vv), k, _ptr(deficient),
            C.byref(ndef), _ptr(stages)))
        return u, s, vv, tuple(int(x) for x in deficient[: ndef.value]), stages

    def rsvd_csr_dev(self, m, n, nnz, rowptr_ptr, col_ptr, val_ptr, k, p, q, seed, u_ptr, s_ptr,
                     v_ptr):
        deficient = np.zeros(max(k + p, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES)
        _check(self.lib.xb_rsvd_csr_dev(
            self.h, m, n, nnz, C.c_void_p(rowptr_ptr), C.c_void_p(col_ptr), C.c_void_p(val_ptr),
            None, int(seed) & (2**64 - 1), k, p, q, C.c_void_p(u_ptr), k, C.c_void_p(s_ptr),
            C.c_void_p(v_ptr), k, _ptr(deficient), C.byref(ndef), _ptr(stages)))
        return tuple(int(x) for x in deficient[: ndef.value]), stages

    def rsvd_csr_sharded_dev(self, m_global, n, m_local, nnz, rowptr_ptr, col_ptr, val_ptr, k, p,
                             q, seed, u_ptr, s_ptr, v_ptr):
        """Row-sharded CSR factorisation (this rank's rows; xb_rsvd_csr_sharded_dev)."""
        deficient = np.zeros(max(k + p, 1), dtype=np.int32)
        ndef = C.c_int(0)
        stages = np.zeros(NUM_STAGES)
        _check(self.lib.xb_rsvd_csr_sharded_dev(
            self.h, m_global, n, m_local, nnz, C.c_void_p(rowptr_ptr), C.c_void_p(col_ptr),
            C.c_void_p(val_ptr), int(seed) & (2**64 - 1), k, p, q, C.c_void_p(u_ptr), k,
            C.c_void_p(s_ptr), C.c_void_p(v_ptr), k, _ptr(deficient), C.byref(ndef),
            _ptr(stages)))
        return tuple(int(x) for x in deficient[: ndef.value]), stages

    def spmm(self, rows, cols, vals, shape, x, trans=False):
        """op(A) @ x for a COO A on the device (xb_spmm_coo)."""
        m, n = shape
        r, c, v = self._coo(rows, cols, vals)
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.ndim != 2 or x.shape[0] != (m if trans else n):
            from .errors import ShapeError

            raise ShapeError(f"inner dimensions disagree: {'A^T' if trans else 'A'} {shape} x {x.shape}")
        out = np.empty((n if trans else m, x.shape[1]))
        _check(self.lib.xb_spmm_coo(self.h, m, n, len(v), _ptr(r), _ptr(c), _ptr(v), int(trans),
                                    _ptr(x), x.shape[1], _ptr(out)))
        return out

    # -- step-level operators -------------------------------------------------------
    def gaussian(self, seed, row0, rows, cols, dtype=np.float64):
        out = np.empty((rows, cols), dtype=dtype)
        _check(self.lib.xb_gaussian(self.h, dtype_code(dtype), int(seed) & (2**64 - 1), row0,
                                    rows, cols, _ptr(out), cols))
        return out

    def uniform_bits(self, seed, row0, rows, cols):
        count = 2 * ((cols + 1) // 2)
        out = np.empty((rows, count), dtype=np.uint64)
        _check(self.lib.xb_uniform_bits(self.h, int(seed) & (2**64 - 1), row0, rows, cols,
                                        _ptr(out)))
        return out

    def gemm(self, a: np.ndarray, b: np.ndarray, trans_a: bool = False):
        """op(a) @ b on the device; a, b host arrays of one dtype."""
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b, dtype=a.dtype)
        if trans_a:
            kdim, m = a.shape
        else:
            m, kdim = a.shape
        if b.shape[0] != kdim:
            from .errors import ShapeError

            raise ShapeError(f"inner dimensions disagree: {a.shape} x {b.shape}")
        n = b.shape[1]
        c = np.empty((m, n), dtype=a.dtype)
        _check(self.lib.xb_gemm(self.h, dtype_code(a.dtype), int(trans_a), m, n, kdim, _ptr(a),
                                a.shape[1], _ptr(b), max(n, 1), _ptr(c), max(n, 1)))
        return c

    def gemm_dev(self, dtype, trans_a, m, n, kdim, a_ptr, lda, b_ptr, ldb, c_ptr, ldc):
        _check(self.lib.xb_gemm_dev(self.h, dtype_code(dtype), int(trans_a), m, n, kdim,
                                    C.c_void_p(a_ptr), lda, C.c_void_p(b_ptr), ldb,
                                    C.c_void_p(c_ptr), ldc))

    def thin_qr(self, y: np.ndarray):
        y = np.ascontiguousarray(y)
        m, r = y.shape
        q = np.empty((m, r), dtype=y.dtype)
        rr = np.empty((r, r), dtype=np.float64)
        deficient = np.zeros(max(r, 1), dtype=np.int32)
        ndef = C.c_int(0)
        _check(self.lib.xb_thin_qr(self.h, dtype_code(y.dtype), m, r, _ptr(y), r, _ptr(q), r,
                                   _ptr(rr), _ptr(deficient), C.byref(ndef)))
        return q, rr, tuple(int(x) for x in deficient[: ndef.value])

    def tsqr_dev(self, m, r, y_ptr, ldy, q_ptr, ldq, r_ptr, ldr):
        """TSQR of a device Y (m x r f64, row-major) into device Q, R
        (xb_tsqr_dev). Returns (deficient columns, device seconds)."""
        deficient = np.zeros(max(r, 1), dtype=np.int32)
        ndef = C.c_int(0)
        sec = np.zeros(1)
        _check(self.lib.xb_tsqr_dev(self.h, m, r, y_ptr, ldy, q_ptr, ldq, r_ptr, ldr,
                                    _ptr(deficient), C.byref(ndef), _ptr(sec)))
        return tuple(int(x) for x in deficient[: ndef.value]), float(sec[0])

    def comm_init_host(self, world: int, rank: int, collective):
        """Host-callback communicator: collective(op, buf) runs the caller's
        collective on the float64 numpy array `buf` in place — op 0: sum over
        ranks; op 1: all-gather (buf = world equal slices, this rank's
        filled). Raises are reported to the library as a failed collective."""

        def tramp(user, op, buf, count):
            try:
                n = int(count) * (world if op == COLL_ALLGATHER else 1)
                arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_double)), shape=(n,))
                collective(int(op), arr)
                return 0
            except BaseException:  # noqa: BLE001 - reported as a status code
                import traceback

                traceback.print_exc()
                return 1

        self._host_coll = HOST_COLLECTIVE(tramp)  # keep the trampoline alive
        _check(self.lib.xb_comm_init_host(self.h, world, rank, self._host_coll, None))

    def svd_small(self, b: np.ndarray):
        b = np.ascontiguousarray(b, dtype=np.float64)
        r, n = b.shape
        u = np.empty((r, r))
        s = np.empty(r)
        v = np.empty((n, r))
        _check(self.lib.xb_svd_small(self.h, r, n, _ptr(b), n, _ptr(u), _ptr(s), _ptr(v)))
        return u, s, v


def load(device: int | None = None) -> Context:
    """The (cached) context for `device` (default: LOCAL_RANK or 0)."""
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    with _lock:
        ctx = _ctxs.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _ctxs[device] = ctx
    return ctx
