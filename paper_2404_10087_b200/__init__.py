"""B200-native FastTuckerPlus engine (arXiv 2404.10087) -- Python binding.

The product is native code: ``libftkcu.so`` (sm_100a kernels + the C-ABI in
``include/ftkcu.h``) and ``libftk.so`` (the drop-in ``ftk::`` C++ API in
``include/ftk/*.hpp``).  This module is a thin ctypes layer over the C-ABI so
tests and ``bench.py`` can drive the engine from Python with numpy buffers.
There is no Python or CPU fallback: if the shared library is missing or no
sm_100 device is present, calls raise ``FtkError``.

Reference counterparts (``/root/reference/proj``): ``ftk::epoch_plus``
(decomposition.cpp:623-705) = :meth:`Session.factor_phase` +
:meth:`Session.core_phase`; ``ftk::loss`` / ``ftk::evaluate``
(evaluation.cpp:36-72) = :meth:`Session.eval`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import host  # noqa: F401  (seed derivation, sampler, counters)

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libftkcu.so")
CXX_LIB_PATH = os.path.join(PKG, "libftk.so")

MODE_DETERMINISTIC = 0
MODE_HOGWILD = 1
PREC_FP32, PREC_TF32, PREC_3XTF32 = 0, 1, 2
EVAL_EXACT, EVAL_FAST = 0, 1
# sweep kernel ids (FTKCU_K_*), read back through get_option("last_factor_kernel")
K_NONE, K_DET, K_WS, K_WS16, K_WS_CC, K_WSF, K_WSG, K_BIG, K_TC, K_HOG, K_WS3 = range(11)

# Every entry point declared in include/ftkcu.h (checked by tests/test_abi.py).
EXPORTS = (
    "ftkcu_abi_version", "ftkcu_session_create", "ftkcu_session_destroy",
    "ftkcu_last_error", "ftkcu_set_option", "ftkcu_get_option", "ftkcu_tensor_upload",
    "ftkcu_tensor_upload_async",
    "ftkcu_tensor_release", "ftkcu_tensor_nnz", "ftkcu_model_upload",
    "ftkcu_model_download", "ftkcu_factor_phase", "ftkcu_core_phase", "ftkcu_eval",
    "ftkcu_batch_probe", "ftkcu_comm_unique_id", "ftkcu_comm_init",
    "ftkcu_comm_allreduce_grad", "ftkcu_tensor_set_cells", "ftkcu_factor_phase_cell",
    "ftkcu_comm_sendrecv_rows", "ftkcu_comm_bcast_rows", "ftkcu_comm_allreduce_f64",
    "ftkcu_stream_sync", "ftkcu_dsgd_factor_epoch", "ftkcu_fasttucker_factor",
    "ftkcu_fasttucker_core", "ftkcu_ccache_upload", "ftkcu_ccache_download",
    "ftkcu_fastertucker_factor", "ftkcu_fastertucker_core", "ftkcu_writeback_ceiling",
    "ftkcu_ring_export", "ftkcu_ring_connect", "ftkcu_ring_emulate", "ftkcu_ring_factor_epoch",
    "ftkcu_ring_status", "ftkcu_ring_debug", "ftkcu_key_layout", "ftkcu_pack_keys",
    "ftkcu_tensor_upload_packed_async", "ftkcu_model_copy_async", "ftkcu_pack_delta",
    "ftkcu_tensor_upload_delta_async",
)


class FtkError(RuntimeError):
    """Mirror of ftk::Error (common.hpp:23-32): every failure raises."""


_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_fpp = C.POINTER(_f32p)

_lib = None


def load_library(path: str = LIB_PATH):
    """Loads libftkcu.so once; raises FtkError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FtkError(f"{path} not built -- run __graft_entry__.build() or make -C {PKG}")
    L = C.CDLL(path)
    L.ftkcu_abi_version.restype = C.c_int
    L.ftkcu_last_error.restype = C.c_char_p
    L.ftkcu_last_error.argtypes = [C.c_void_p]
    L.ftkcu_session_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.ftkcu_session_destroy.argtypes = [C.c_void_p]
    L.ftkcu_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
    L.ftkcu_get_option.argtypes = [C.c_void_p, C.c_char_p, _i64p]
    L.ftkcu_tensor_upload.argtypes = [C.c_void_p, C.c_int, C.c_int, _i32p, C.c_int64, _i32p,
                                      _f32p]
    L.ftkcu_tensor_upload_async.argtypes = [C.c_void_p, C.c_int, C.c_int, _i32p, C.c_int64,
                                            _i32p, _f32p]
    L.ftkcu_fasttucker_factor.argtypes = [C.c_void_p, C.c_int, C.c_int, _i64p, _i64p, C.c_int64,
                                          C.c_int32, C.c_float, C.c_float, _f64p]
    L.ftkcu_fasttucker_core.argtypes = [C.c_void_p, C.c_int, C.c_int, _i64p, C.c_int32,
                                        C.c_float, C.c_float, C.c_int, _f64p]
    L.ftkcu_ccache_upload.argtypes = [C.c_void_p, _fpp]
    L.ftkcu_ccache_download.argtypes = [C.c_void_p, _fpp]
    L.ftkcu_fastertucker_factor.argtypes = [C.c_void_p, C.c_int, C.c_int, _i64p, _i64p,
                                            C.c_int64, C.c_float, C.c_float, _f64p]
    L.ftkcu_fastertucker_core.argtypes = [C.c_void_p, C.c_int, C.c_int, _i64p, _i64p,
                                          C.c_int64, C.c_float, C.c_float, C.c_int, _f64p]
    L.ftkcu_tensor_release.argtypes = [C.c_void_p, C.c_int]
    L.ftkcu_tensor_nnz.argtypes = [C.c_void_p, C.c_int]
    L.ftkcu_tensor_nnz.restype = C.c_int64
    L.ftkcu_model_upload.argtypes = [C.c_void_p, C.c_int, _i32p, _i32p, C.c_int32, _fpp, _fpp]
    L.ftkcu_model_download.argtypes = [C.c_void_p, _fpp, _fpp]
    L.ftkcu_factor_phase.argtypes = [C.c_void_p, C.c_int, _i64p, C.c_int32, C.c_float,
                                     C.c_float, C.c_int, C.c_uint64, _f64p]
    L.ftkcu_core_phase.argtypes = [C.c_void_p, C.c_int, _i64p, C.c_int32, C.c_float,
                                   C.c_float, C.c_int, C.c_uint64, _f32p, _f64p]
    L.ftkcu_eval.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_double, _f64p]
    L.ftkcu_batch_probe.argtypes = [C.c_void_p, C.c_int, _i64p, C.c_int, C.c_int, C.c_float,
                                    C.c_float] + [_f32p] * 9
    L.ftkcu_comm_unique_id.argtypes = [C.c_char_p]
    L.ftkcu_comm_init.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int]
    L.ftkcu_comm_allreduce_grad.argtypes = [C.c_void_p]
    L.ftkcu_tensor_set_cells.argtypes = [C.c_void_p, C.c_int, _i64p, C.c_int]
    L.ftkcu_factor_phase_cell.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_float,
                                          C.c_uint64, _f64p]
    L.ftkcu_comm_sendrecv_rows.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int,
                                           C.c_int64, C.c_int64, C.c_int]
    L.ftkcu_comm_bcast_rows.argtypes = [C.c_void_p, C.c_int, _i64p, C.c_int]
    L.ftkcu_comm_allreduce_f64.argtypes = [C.c_void_p, _f64p, C.c_int]
    L.ftkcu_stream_sync.argtypes = [C.c_void_p]
    L.ftkcu_writeback_ceiling.argtypes = [C.c_void_p, C.c_int, C.c_uint64, _f64p]
    L.ftkcu_dsgd_factor_epoch.argtypes = [C.c_void_p, C.c_int, C.c_int, _i64p, _i64p,
                                          C.POINTER(C.c_uint64), C.c_float, C.c_float, _f64p]
    L.ftkcu_ring_export.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
    L.ftkcu_ring_connect.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int]
    L.ftkcu_ring_emulate.argtypes = [C.c_void_p, C.c_int]
    L.ftkcu_ring_factor_epoch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, _i64p, _i64p,
                                          C.POINTER(C.c_uint64), C.c_float, C.c_float, _f64p]
    L.ftkcu_ring_status.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
    L.ftkcu_key_layout.argtypes = [C.c_int, _i32p, C.POINTER(C.c_int)]
    L.ftkcu_model_copy_async.argtypes = [C.c_void_p, C.c_int, _fpp, _fpp]
    L.ftkcu_pack_keys.argtypes = [C.c_int, _i32p, C.c_int64, _i32p, C.POINTER(C.c_uint32),
                                  C.c_void_p]
    L.ftkcu_tensor_upload_packed_async.argtypes = [C.c_void_p, C.c_int, C.c_int, _i32p,
                                                   C.c_int64, C.POINTER(C.c_uint32), C.c_void_p,
                                                   _f32p]
    L.ftkcu_pack_delta.argtypes = [C.c_int, _i32p, C.c_int64, _i32p, _f32p, C.c_void_p,
                                   C.c_int64, C.POINTER(C.c_uint64), _f32p, C.POINTER(C.c_int)]
    L.ftkcu_tensor_upload_delta_async.argtypes = [C.c_void_p, C.c_int, C.c_int, _i32p, C.c_int64,
                                                  C.c_void_p, C.c_int, C.POINTER(C.c_uint64),
                                                  _f32p]
    L.ftkcu_ring_debug.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                   C.c_int]
    _lib = L
    return L


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _ptrs(arrs):
    out = (_f32p * len(arrs))()
    for i, a in enumerate(arrs):
        if a.dtype != np.float32 or not a.flags.c_contiguous:
            raise FtkError("model matrices must be C-contiguous float32")
        out[i] = a.ctypes.data_as(_f32p)
    return out


class Session:
    """One engine session on one CUDA device (``ftkcu_session``)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.ftkcu_session_create(device, C.byref(h))
        if rc != 0:
            raise FtkError(self.lib.ftkcu_last_error(None).decode())
        self.h = h
        self.order = 0
        self.ranks = None
        self.r = 0
        self.dims = None

    # -- plumbing
    def _ck(self, rc):
        if rc != 0:
            raise FtkError(self.lib.ftkcu_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.ftkcu_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_option(self, key: str, value: int):
        self._ck(self.lib.ftkcu_set_option(self.h, key.encode(), int(value)))

    def get_option(self, key: str) -> int:
        v = C.c_int64()
        self._ck(self.lib.ftkcu_get_option(self.h, key.encode(), C.byref(v)))
        return v.value

    @property
    def stream_handle(self) -> int:
        """cudaStream_t of the session (for torch.cuda.ExternalStream timing)."""
        return self.get_option("stream")

    # -- data
    def upload_tensor(self, slot, dims, idx, vals):
        dims = np.ascontiguousarray(dims, np.int32)
        idx = np.ascontiguousarray(idx, np.int32)
        vals = np.ascontiguousarray(vals, np.float32)
        nnz = vals.shape[0]
        if idx.shape != (nnz, dims.shape[0]):
            raise FtkError("index array must be nnz x order")
        self._ck(self.lib.ftkcu_tensor_upload(self.h, slot, dims.shape[0], _p(dims, _i32p), nnz,
                                              _p(idx, _i32p), _p(vals, _f32p)))

    def upload_tensor_ptr(self, slot, dims, nnz, idx_ptr: int, vals_ptr: int):
        """Upload from raw (e.g. pinned) host pointers."""
        dims = np.ascontiguousarray(dims, np.int32)
        self._ck(self.lib.ftkcu_tensor_upload(self.h, slot, dims.shape[0], _p(dims, _i32p), nnz,
                                              C.cast(idx_ptr, _i32p), C.cast(vals_ptr, _f32p)))

    def upload_tensor_ptr_async(self, slot, dims, nnz, idx_ptr: int, vals_ptr: int):
        """Asynchronous upload from pinned host pointers (copy stream); the
        slot's next use waits for it.  The host buffers must stay alive."""
        dims = np.ascontiguousarray(dims, np.int32)
        self._ck(self.lib.ftkcu_tensor_upload_async(self.h, slot, dims.shape[0],
                                                    _p(dims, _i32p), nnz, C.cast(idx_ptr, _i32p),
                                                    C.cast(vals_ptr, _f32p)))

    @staticmethod
    def pack_keys(dims, idx):
        """Packed-key COO (ftkcu_pack_keys): every mode's index in one bit
        field per nonzero, as (lo uint32 array, hi uint16/uint32 array or
        None); 10 bytes per nonzero with the values at the Netflix shape
        instead of 16 on the host-to-device link."""
        L = load_library()
        dims = np.ascontiguousarray(dims, np.int32)
        idx = np.ascontiguousarray(idx, np.int32)
        hb = C.c_int(0)
        if L.ftkcu_key_layout(dims.shape[0], _p(dims, _i32p), C.byref(hb)) != 0:
            raise FtkError(L.ftkcu_last_error(None).decode())
        lo = np.empty(idx.shape[0], np.uint32)
        hi = np.empty(idx.shape[0], {2: np.uint16, 4: np.uint32}[hb.value]) if hb.value else None
        rc = L.ftkcu_pack_keys(dims.shape[0], _p(dims, _i32p), idx.shape[0], _p(idx, _i32p),
                               lo.ctypes.data_as(C.POINTER(C.c_uint32)),
                               None if hi is None else hi.ctypes.data)
        if rc != 0:
            raise FtkError(L.ftkcu_last_error(None).decode())
        return lo, hi

    @staticmethod
    def pack_delta(dims, idx, vals):
        """Delta-coded COO (ftkcu_pack_delta): the nonzeros sorted by their
        mixed-radix key, as (deltas uint8 [width * nnz], restarts uint64
        [ceil(nnz / 4096)], values float32 in the sorted order, width)."""
        L = load_library()
        dims = np.ascontiguousarray(dims, np.int32)
        idx = np.ascontiguousarray(idx, np.int32)
        vals = np.ascontiguousarray(vals, np.float32)
        nnz = idx.shape[0]
        restarts = np.empty((nnz + 4095) // 4096, np.uint64)
        vout = np.empty(nnz, np.float32)
        w = C.c_int(0)
        for cap in (4, 8):
            deltas = np.empty(cap * nnz, np.uint8)
            rc = L.ftkcu_pack_delta(dims.shape[0], _p(dims, _i32p), nnz, _p(idx, _i32p),
                                    _p(vals, _f32p), deltas.ctypes.data, deltas.size,
                                    restarts.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    _p(vout, _f32p), C.byref(w))
            if rc == 0:
                return deltas[:w.value * nnz], restarts, vout, w.value
            if w.value <= cap:
                break
        raise FtkError(L.ftkcu_last_error(None).decode())

    def upload_tensor_delta_ptr_async(self, slot, dims, nnz, deltas_ptr: int, width: int,
                                      restarts_ptr: int, vals_ptr: int):
        """ftkcu_tensor_upload_delta_async from pinned host pointers."""
        dims = np.ascontiguousarray(dims, np.int32)
        self._ck(self.lib.ftkcu_tensor_upload_delta_async(
            self.h, slot, dims.shape[0], _p(dims, _i32p), nnz, deltas_ptr, width,
            C.cast(restarts_ptr, C.POINTER(C.c_uint64)), C.cast(vals_ptr, _f32p)))

    def upload_tensor_packed_ptr_async(self, slot, dims, nnz, lo_ptr: int, hi_ptr, vals_ptr: int):
        """ftkcu_tensor_upload_packed_async from pinned host pointers
        (hi_ptr None when the keys have no high part)."""
        dims = np.ascontiguousarray(dims, np.int32)
        self._ck(self.lib.ftkcu_tensor_upload_packed_async(
            self.h, slot, dims.shape[0], _p(dims, _i32p), nnz,
            C.cast(lo_ptr, C.POINTER(C.c_uint32)), hi_ptr, C.cast(vals_ptr, _f32p)))

    def model_copy_async(self, to_device: bool, a, b):
        """Enqueued model upload (to_device) or download into pinned numpy
        views a[n], b[n]; completes in stream order (sync() waits)."""
        ap = (_f32p * len(a))(*[x.ctypes.data_as(_f32p) for x in a])
        bp = (_f32p * len(b))(*[x.ctypes.data_as(_f32p) for x in b])
        self._ck(self.lib.ftkcu_model_copy_async(self.h, 1 if to_device else 0, ap, bp))

    def release_tensor(self, slot):
        self._ck(self.lib.ftkcu_tensor_release(self.h, slot))

    def upload_model(self, dims, ranks, r, a, b):
        dims = np.ascontiguousarray(dims, np.int32)
        ranks = np.ascontiguousarray(ranks, np.int32)
        self._ck(self.lib.ftkcu_model_upload(self.h, dims.shape[0], _p(dims, _i32p),
                                             _p(ranks, _i32p), int(r), _ptrs(a), _ptrs(b)))
        self.order, self.dims, self.ranks, self.r = dims.shape[0], dims.copy(), ranks.copy(), int(r)

    def download_model(self, a=None, b=None):
        if a is None:
            a = [np.empty((int(d), int(j)), np.float32) for d, j in zip(self.dims, self.ranks)]
        if b is None:
            b = [np.empty((int(j), self.r), np.float32) for j in self.ranks]
        self._ck(self.lib.ftkcu_model_download(self.h, _ptrs(a), _ptrs(b)))
        return a, b

    # -- hot path
    def factor_phase(self, slot=0, perm=None, M=16, lr_a=1e-3, reg_a=1e-4,
                     mode=MODE_DETERMINISTIC, seed=0, timed=True):
        pa = None if perm is None else np.ascontiguousarray(perm, np.int64)
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_factor_phase(self.h, slot, _p(pa, _i64p), M, lr_a, reg_a, mode,
                                             C.c_uint64(seed & (2**64 - 1)),
                                             C.byref(ms) if timed else None))
        return ms.value

    def core_phase(self, slot=0, perm=None, M=16, lr_b=1e-3, reg_b=1e-4,
                   mode=MODE_DETERMINISTIC, seed=0, want_grad=False, timed=True):
        pa = None if perm is None else np.ascontiguousarray(perm, np.int64)
        g = np.zeros(int(np.sum(self.ranks)) * self.r, np.float32) if want_grad else None
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_core_phase(self.h, slot, _p(pa, _i64p), M, lr_b, reg_b, mode,
                                           C.c_uint64(seed & (2**64 - 1)), _p(g, _f32p),
                                           C.byref(ms) if timed else None))
        return (ms.value, g) if want_grad else ms.value

    def fasttucker_factor(self, slot, mode, perm, bucket_off, M=16, lr_a=1e-3, reg_a=1e-4,
                          timed=True):
        """FastTucker factor block of `mode` over a per-bucket plan
        (ftkcu_fasttucker_factor)."""
        pa = np.ascontiguousarray(perm, np.int64)
        bo = np.ascontiguousarray(bucket_off, np.int64)
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_fasttucker_factor(self.h, slot, mode, _p(pa, _i64p), _p(bo, _i64p),
                                                  bo.size - 1, M, lr_a, reg_a,
                                                  C.byref(ms) if timed else None))
        return ms.value

    def fasttucker_core(self, slot, mode, perm, M=16, lr_b=1e-3, reg_b=1e-4,
                        schedule=MODE_DETERMINISTIC, timed=True):
        """FastTucker core block of `mode` over a global plan (ftkcu_fasttucker_core)."""
        pa = np.ascontiguousarray(perm, np.int64)
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_fasttucker_core(self.h, slot, mode, _p(pa, _i64p), M, lr_b,
                                                reg_b, schedule, C.byref(ms) if timed else None))
        return ms.value

    def ccache_upload(self, cache):
        """The FasterTucker C cache (list of dims[n] x R fp32 arrays) to the device."""
        cs = [np.ascontiguousarray(c, np.float32) for c in cache]
        self._ck(self.lib.ftkcu_ccache_upload(self.h, _ptrs(cs)))

    def ccache_download(self):
        out = [np.empty((int(d), self.r), np.float32) for d in self.dims]
        self._ck(self.lib.ftkcu_ccache_download(self.h, _ptrs(out)))
        return out

    def fastertucker_factor(self, slot, mode, perm, row_off, lr_a=1e-3, reg_a=1e-4, timed=True):
        pa = np.ascontiguousarray(perm, np.int64)
        ro = np.ascontiguousarray(row_off, np.int64)
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_fastertucker_factor(self.h, slot, mode, _p(pa, _i64p),
                                                    _p(ro, _i64p), ro.size - 1, lr_a, reg_a,
                                                    C.byref(ms) if timed else None))
        return ms.value

    def fastertucker_core(self, slot, mode, perm, batch_off, lr_b=1e-3, reg_b=1e-4,
                          schedule=MODE_DETERMINISTIC, timed=True):
        pa = np.ascontiguousarray(perm, np.int64)
        bo = np.ascontiguousarray(batch_off, np.int64)
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_fastertucker_core(self.h, slot, mode, _p(pa, _i64p),
                                                  _p(bo, _i64p), bo.size - 1, lr_b, reg_b,
                                                  schedule, C.byref(ms) if timed else None))
        return ms.value

    def eval(self, slot=1, workers=1, reg_a=0.0, reg_b=0.0):
        out = np.zeros(3, np.float64)
        self._ck(self.lib.ftkcu_eval(self.h, slot, workers, reg_a, reg_b, _p(out, _f64p)))
        return out

    def batch_probe(self, slot, rows, cap, lr_a, reg_a):
        rows = np.ascontiguousarray(rows, np.int64)
        order, r, jmax = self.order, self.r, int(np.max(self.ranks))
        out = dict(
            c=np.zeros((order, cap, r), np.float32), d=np.zeros((order, cap, r), np.float32),
            u=np.zeros((order, cap, jmax), np.float32), xhat_f=np.zeros(cap, np.float32),
            resid_f=np.zeros(cap, np.float32), xhat_c=np.zeros(cap, np.float32),
            resid_c=np.zeros(cap, np.float32), a_new=np.zeros((order, cap, jmax), np.float32),
            g=np.zeros((order, jmax, r), np.float32))
        self._ck(self.lib.ftkcu_batch_probe(
            self.h, slot, _p(rows, _i64p), rows.size, cap, lr_a, reg_a,
            *[_p(out[k], _f32p) for k in ("c", "d", "u", "xhat_f", "resid_f", "xhat_c",
                                           "resid_c", "a_new", "g")]))
        return out

    # -- multi-GPU
    @staticmethod
    def comm_unique_id() -> bytes:
        L = load_library()
        buf = C.create_string_buffer(128)
        rc = L.ftkcu_comm_unique_id(buf)
        if rc != 0:
            raise FtkError(L.ftkcu_last_error(None).decode())
        return buf.raw

    def comm_init(self, uid: bytes, rank: int, world: int):
        self._ck(self.lib.ftkcu_comm_init(self.h, uid, rank, world))

    # -- DSGD strata (paper_2404_10087_b200/dsgd.py drives these)
    def set_cells(self, slot, cell_offsets):
        off = np.ascontiguousarray(cell_offsets, np.int64)
        self._ck(self.lib.ftkcu_tensor_set_cells(self.h, slot, _p(off, _i64p), off.size - 1))

    def factor_phase_cell(self, slot, cell, lr_a=1e-3, reg_a=1e-4, seed=0, timed=False):
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_factor_phase_cell(self.h, slot, cell, lr_a, reg_a,
                                                  C.c_uint64(seed & (2**64 - 1)),
                                                  C.byref(ms) if timed else None))
        return ms.value

    def sendrecv_rows(self, mode, send_row0, send_nrows, dst, recv_row0, recv_nrows, src):
        self._ck(self.lib.ftkcu_comm_sendrecv_rows(self.h, mode, send_row0, send_nrows, dst,
                                                   recv_row0, recv_nrows, src))

    def bcast_rows(self, mode, row_off):
        off = np.ascontiguousarray(row_off, np.int64)
        self._ck(self.lib.ftkcu_comm_bcast_rows(self.h, mode, _p(off, _i64p), off.size - 1))

    def allreduce_f64(self, values):
        v = np.ascontiguousarray(values, np.float64).copy()
        self._ck(self.lib.ftkcu_comm_allreduce_f64(self.h, _p(v, _f64p), v.size))
        return v

    def dsgd_factor_epoch(self, slot, parts, row_off2, row_off3, cell_seeds, lr_a=1e-3,
                          reg_a=1e-4, timed=False):
        o2 = np.ascontiguousarray(row_off2, np.int64)
        o3 = np.ascontiguousarray(row_off3, np.int64)
        sd = np.ascontiguousarray(np.asarray(cell_seeds, np.uint64))
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_dsgd_factor_epoch(
            self.h, slot, parts, _p(o2, _i64p), _p(o3, _i64p), _p(sd, C.POINTER(C.c_uint64)),
            lr_a, reg_a, C.byref(ms) if timed else None))
        return ms.value

    # -- DSGD ring epochs (token-passing mode-3 blocks; dsgd.RingTrainer)
    RING_BLOB_BYTES = 512

    def ring_export(self) -> bytes:
        """This session's peer descriptor (factor matrices + arrival flags)."""
        buf = C.create_string_buffer(self.RING_BLOB_BYTES)
        self._ck(self.lib.ftkcu_ring_export(self.h, buf, self.RING_BLOB_BYTES))
        return buf.raw

    def ring_connect(self, slot, left_blob: bytes):
        """Maps the left neighbour's (rank - 1) descriptor, clears this rank's
        flags and prepares `slot` (uploaded, cells set) for ring epochs."""
        self._ck(self.lib.ftkcu_ring_connect(self.h, slot, left_blob, len(left_blob)))

    def ring_emulate(self, slot):
        """No peers: posts go to local scratch and waits are skipped (timing)."""
        self._ck(self.lib.ftkcu_ring_emulate(self.h, slot))

    def ring_factor_epoch(self, slot, parts, rank, row_off2, row_off3, cell_seeds, lr_a=1e-3,
                          reg_a=1e-4, timed=False):
        o2 = np.ascontiguousarray(row_off2, np.int64)
        o3 = np.ascontiguousarray(row_off3, np.int64)
        sd = np.ascontiguousarray(np.asarray(cell_seeds, np.uint64))
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_ring_factor_epoch(
            self.h, slot, parts, rank, _p(o2, _i64p), _p(o3, _i64p),
            _p(sd, C.POINTER(C.c_uint64)), lr_a, reg_a, C.byref(ms) if timed else None))
        return ms.value

    def ring_status(self) -> int:
        """Synchronises; nonzero if a ring wait timed out (the epoch is
        invalid): 0x10000 | flag id of the first stuck block wait, or
        0x20000 | round of a stuck post (a block copy waiting for its cell)."""
        v = C.c_int(0)
        self._ck(self.lib.ftkcu_ring_status(self.h, C.byref(v)))
        return int(v.value)

    def ring_debug(self, n):
        """(arrival flags, cell counters), first n entries each (tests)."""
        f = np.zeros(n, np.uint32)
        d = np.zeros(n, np.uint32)
        self._ck(self.lib.ftkcu_ring_debug(self.h, f.ctypes.data_as(C.POINTER(C.c_uint32)),
                                           d.ctypes.data_as(C.POINTER(C.c_uint32)), n))
        return f, d

    def sync(self):
        self._ck(self.lib.ftkcu_stream_sync(self.h))

    def writeback_ceiling(self, slot=0, seed=0) -> float:
        """Device ms of the J = R = 32 factor sweep's RED write-back alone over
        slot's tile stream (measurement; the model is untouched)."""
        ms = C.c_double(0.0)
        self._ck(self.lib.ftkcu_writeback_ceiling(self.h, slot, C.c_uint64(seed & (2**64 - 1)),
                                                  C.byref(ms)))
        return ms.value
