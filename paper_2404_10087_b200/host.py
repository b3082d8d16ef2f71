"""ctypes wrapper of ``libftk.so`` -- the drop-in ``ftk::`` C++ API.

These calls run the engine's C++ host layer (``paper_2404_10087_b200/host``):
the libstdc++-exact sampler / split / init, and ``ftk::epoch_plus`` /
``ftk::train`` / ``ftk::loss`` / ``ftk::evaluate`` on the device.  Numpy
arrays in, numpy arrays out.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libftk.so")

M64 = (1 << 64) - 1

_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_fpp = C.POINTER(_f32p)

_lib = None


class HostError(RuntimeError):
    pass


def mix64(x: int) -> int:
    """splitmix64 step (reference common.hpp:35-41), pure Python."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def derive_seed(base: int, path) -> int:
    """derive_seed(base, {path...}) (reference common.hpp:44-48)."""
    s = mix64(base & M64)
    for p in path:
        s = mix64(s ^ (p & M64))
    return s


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise HostError(f"{LIB_PATH} not built")
    L = C.CDLL(LIB_PATH)
    L.ftkh_last_error.restype = C.c_char_p
    L.ftkh_derive_seed.restype = C.c_uint64
    L.ftkh_derive_seed.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_int]
    L.ftkh_global_plan.argtypes = [C.c_int64, C.c_int, C.c_uint64, _i64p]
    L.ftkh_per_bucket_plan.argtypes = [C.c_int, C.c_int64, _i32p, C.c_int, C.c_int, C.c_int,
                                       C.c_uint64, _i64p, _i64p, _i64p]
    L.ftkh_init_model.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_uint64, C.c_float, _fpp,
                                  _fpp]
    L.ftkh_default_init_scale.restype = C.c_float
    L.ftkh_default_init_scale.argtypes = [C.c_double, C.c_int, C.c_int32, _i32p]
    L.ftkh_split.argtypes = [C.c_int, _i32p, C.c_int64, _i32p, _f32p, C.c_double, C.c_uint64,
                             _i32p, _f32p, _i32p, _f32p, _i64p]
    L.ftkh_load_coo.restype = C.c_void_p
    L.ftkh_load_coo.argtypes = [C.c_char_p, C.c_int]
    L.ftkh_infer_coo_order.argtypes = [C.c_char_p]
    L.ftkh_tensor_nnz.restype = C.c_int64
    L.ftkh_tensor_nnz.argtypes = [C.c_void_p]
    L.ftkh_tensor_copy.argtypes = [C.c_void_p, _i32p, _i32p, _f32p]
    L.ftkh_tensor_free.argtypes = [C.c_void_p]
    L.ftkh_save_coo.argtypes = [C.c_int, _i32p, C.c_int64, _i32p, _f32p, C.c_char_p]
    L.ftkh_load_coo_binary.restype = C.c_void_p
    L.ftkh_load_coo_binary.argtypes = [C.c_char_p]
    L.ftkh_tensor_order.argtypes = [C.c_void_p]
    L.ftkh_save_coo_binary.argtypes = [C.c_int, _i32p, C.c_int64, _i32p, _f32p, C.c_char_p]
    L.ftkh_set_device_options.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
    L.ftkh_epoch_plus.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_int64, _i32p, _f32p,
                                  _fpp, _fpp, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int,
                                  C.c_int, C.c_int, C.c_int, C.c_uint64, _f64p, _i64p]
    L.ftkh_epoch_fasttucker.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_int64, _i32p,
                                        _f32p, _fpp, _fpp, C.c_float, C.c_float, C.c_float,
                                        C.c_float, C.c_int, C.c_int, C.c_int, C.c_uint64, _f64p,
                                        _i64p]
    L.ftkh_epoch_fastertucker.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_int64, _i32p,
                                          _f32p, _fpp, _fpp, C.c_float, C.c_float, C.c_float,
                                          C.c_float, C.c_int, C.c_int, C.c_int, C.c_uint64, _f64p,
                                          _i64p]
    L.ftkh_train.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_int64, _i32p, _f32p,
                             C.c_int64, _i32p, _f32p, _fpp, _fpp, C.c_float, C.c_float,
                             C.c_float, C.c_float, C.c_int, C.c_int, C.c_int, C.c_int,
                             C.c_uint64, _f64p, _f64p, _f64p, _f64p, _i64p, _i64p, C.c_char_p,
                             C.c_int]
    L.ftkh_train_variant.argtypes = list(L.ftkh_train.argtypes) + [C.c_int]
    L.ftkh_loss.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_int64, _i32p, _f32p, _fpp,
                            _fpp, C.c_double, C.c_double, C.c_int, _f64p]
    L.ftkh_evaluate.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_int64, _i32p, _f32p, _fpp,
                                _fpp, C.c_int, _f64p, _f64p]
    L.ftkh_predicted_costs.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i64p]
    _lib = L
    return L


def _ck(rc):
    if rc != 0:
        raise HostError(lib().ftkh_last_error().decode())


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _ptrs(arrs):
    out = (_f32p * len(arrs))()
    for i, a in enumerate(arrs):
        assert a.dtype == np.float32 and a.flags.c_contiguous
        out[i] = a.ctypes.data_as(_f32p)
    return out


def _i32(a):
    return np.ascontiguousarray(a, np.int32)


def global_plan(nnz: int, m: int, seed: int) -> np.ndarray:
    """EpochPlan::global positions for Rng(seed) (libstdc++ std::shuffle)."""
    out = np.empty(nnz, np.int64)
    _ck(lib().ftkh_global_plan(nnz, m, seed & M64, _p(out, _i64p)))
    return out


def per_bucket_plan(idx, mode: int, m: int, seed: int, keying: int = 0):
    """EpochPlan::per_bucket over build_mode_index(mode, keying) for Rng(seed):
    (positions in plan order, bucket offsets in plan order incl. nnz).
    keying 0 = fixed mode (FastTucker), 1 = fixed complement."""
    idx = np.ascontiguousarray(idx, np.int32)
    nnz, order = idx.shape
    perm = np.empty(nnz, np.int64)
    boff = np.empty(nnz + 2, np.int64)
    nb = C.c_int64(0)
    _ck(lib().ftkh_per_bucket_plan(order, nnz, _p(idx, _i32p), mode, keying, m, seed & M64,
                                   _p(perm, _i64p), _p(boff, _i64p), C.byref(nb)))
    return perm, boff[: nb.value + 1].copy()


def init_model(dims, ranks, r, seed, scale):
    dims, ranks = _i32(dims), _i32(ranks)
    a = [np.empty((int(d), int(j)), np.float32) for d, j in zip(dims, ranks)]
    b = [np.empty((int(j), int(r)), np.float32) for j in ranks]
    _ck(lib().ftkh_init_model(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r, seed & M64, scale,
                              _ptrs(a), _ptrs(b)))
    return a, b


def default_init_scale(mean_abs, order, r, ranks) -> float:
    ranks = _i32(ranks)
    return lib().ftkh_default_init_scale(mean_abs, order, r, _p(ranks, _i32p))


def split_train_test(dims, idx, vals, frac, seed):
    dims, idx = _i32(dims), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    nnz, order = idx.shape
    tr_i = np.empty((nnz, order), np.int32)
    te_i = np.empty((nnz, order), np.int32)
    tr_v = np.empty(nnz, np.float32)
    te_v = np.empty(nnz, np.float32)
    nt = C.c_int64()
    _ck(lib().ftkh_split(order, _p(dims, _i32p), nnz, _p(idx, _i32p), _p(vals, _f32p), frac,
                         seed & M64, _p(tr_i, _i32p), _p(tr_v, _f32p), _p(te_i, _i32p),
                         _p(te_v, _f32p), C.byref(nt)))
    k = nt.value
    return (tr_i[: nnz - k], tr_v[: nnz - k]), (te_i[:k], te_v[:k])


def load_coo(path: str, order: int = 0):
    L = lib()
    if order <= 0:
        order = L.ftkh_infer_coo_order(path.encode())
        if order < 0:
            raise HostError(L.ftkh_last_error().decode())
    h = L.ftkh_load_coo(path.encode(), order)
    if not h:
        raise HostError(L.ftkh_last_error().decode())
    try:
        nnz = L.ftkh_tensor_nnz(h)
        dims = np.empty(order, np.int32)
        idx = np.empty((nnz, order), np.int32)
        vals = np.empty(nnz, np.float32)
        L.ftkh_tensor_copy(h, _p(dims, _i32p), _p(idx, _i32p), _p(vals, _f32p))
        return dims, idx, vals
    finally:
        L.ftkh_tensor_free(h)


def load_coo_binary(path: str):
    """ftk::load_coo_binary (FTKC1): (dims, idx [nnz x order], vals)."""
    L = lib()
    h = L.ftkh_load_coo_binary(path.encode())
    if not h:
        raise HostError(L.ftkh_last_error().decode())
    try:
        order, nnz = L.ftkh_tensor_order(h), L.ftkh_tensor_nnz(h)
        dims = np.empty(order, np.int32)
        idx = np.empty((nnz, order), np.int32)
        vals = np.empty(nnz, np.float32)
        L.ftkh_tensor_copy(h, _p(dims, _i32p), _p(idx, _i32p), _p(vals, _f32p))
        return dims, idx, vals
    finally:
        L.ftkh_tensor_free(h)


def save_coo_binary(dims, idx, vals, path):
    dims, idx = _i32(dims), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    _ck(lib().ftkh_save_coo_binary(dims.size, _p(dims, _i32p), vals.size, _p(idx, _i32p),
                                   _p(vals, _f32p), path.encode()))


def save_coo(dims, idx, vals, path):
    dims, idx = _i32(dims), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    _ck(lib().ftkh_save_coo(dims.size, _p(dims, _i32p), vals.size, _p(idx, _i32p),
                            _p(vals, _f32p), path.encode()))


def set_device_options(device=-1, mode=0, precision=1, exact_eval=True, parity=False):
    """mode 0 auto / 1 deterministic / 2 hogwild; precision 0 fp32 / 1 tf32
    (the C++ default) / 2 3xtf32; parity: Hogwild at the reference's
    asynchrony noise floor (ftk::DeviceOptions::parity)."""
    _ck(lib().ftkh_set_device_options(device, mode, precision, int(exact_eval), int(parity)))


def last_kernels():
    """(factor, core) FTKCU_K_* ids of the sweeps the last ftk:: epoch ran."""
    f, c = C.c_int(0), C.c_int(0)
    _ck(lib().ftkh_last_kernels(C.byref(f), C.byref(c)))
    return f.value, c.value


def epoch_plus(dims, ranks, r, idx, vals, a, b, seed, lr_a=1e-3, lr_b=1e-3, reg_a=1e-4,
               reg_b=1e-4, m=16, workers=1, store_c=False, canonical=False):
    """ftk::epoch_plus through the C++ API; mutates a/b in place."""
    dims, ranks, idx = _i32(dims), _i32(ranks), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    secs = np.zeros(2, np.float64)
    cnt = np.zeros(10, np.int64)
    _ck(lib().ftkh_epoch_plus(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r, vals.size,
                              _p(idx, _i32p), _p(vals, _f32p), _ptrs(a), _ptrs(b), lr_a, lr_b,
                              reg_a, reg_b, m, workers, int(store_c), int(canonical), seed & M64,
                              _p(secs, _f64p), _p(cnt, _i64p)))
    return secs, cnt


def epoch_fasttucker(dims, ranks, r, idx, vals, a, b, seed, lr_a=1e-3, lr_b=1e-3, reg_a=1e-4,
                     reg_b=1e-4, m=16, canonical=False, workers=1):
    """ftk::epoch_fasttucker through the C++ API (fixed-mode indices built
    there); mutates a/b in place; returns (seconds[2], counters[10])."""
    dims, ranks, idx = _i32(dims), _i32(ranks), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    secs = np.zeros(2, np.float64)
    cnt = np.zeros(10, np.int64)
    _ck(lib().ftkh_epoch_fasttucker(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r, vals.size,
                                    _p(idx, _i32p), _p(vals, _f32p), _ptrs(a), _ptrs(b), lr_a,
                                    lr_b, reg_a, reg_b, m, workers, int(canonical), seed & M64,
                                    _p(secs, _f64p), _p(cnt, _i64p)))
    return secs, cnt


def epoch_fastertucker(dims, ranks, r, idx, vals, a, b, seed, lr_a=1e-3, lr_b=1e-3,
                       reg_a=1e-4, reg_b=1e-4, m=16, canonical=False, workers=1):
    """ftk::epoch_fastertucker through the C++ API (complement indices and a
    fresh C cache built there); mutates a/b; returns (seconds[2], counters[10])."""
    dims, ranks, idx = _i32(dims), _i32(ranks), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    secs = np.zeros(2, np.float64)
    cnt = np.zeros(10, np.int64)
    _ck(lib().ftkh_epoch_fastertucker(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r, vals.size,
                                      _p(idx, _i32p), _p(vals, _f32p), _ptrs(a), _ptrs(b), lr_a,
                                      lr_b, reg_a, reg_b, m, workers, int(canonical), seed & M64,
                                      _p(secs, _f64p), _p(cnt, _i64p)))
    return secs, cnt


VARIANTS = {"plus": 0, "fasttucker": 1, "fastertucker": 2}


def train(dims, ranks, r, train_idx, train_vals, test_idx, test_vals, a, b, epochs, seed,
          lr_a=1e-3, lr_b=1e-3, reg_a=1e-4, reg_b=1e-4, m=16, workers=1, store_c=False,
          variant="plus"):
    """ftk::train through the C++ API (TrainOptions.variant); mutates a/b;
    returns per-epoch history."""
    dims, ranks = _i32(dims), _i32(ranks)
    tri, trv = _i32(train_idx), np.ascontiguousarray(train_vals, np.float32)
    if test_idx is None:
        tei, tev, nte = None, None, 0
    else:
        tei, tev = _i32(test_idx), np.ascontiguousarray(test_vals, np.float32)
        nte = tev.size
    out = {k: np.zeros(epochs, np.float64) for k in ("loss", "rmse", "mae", "seconds")}
    reads = np.zeros(epochs, np.int64)
    mults = np.zeros(epochs, np.int64)
    cap = 256 * max(epochs, 1) + 64
    buf = C.create_string_buffer(cap)
    _ck(lib().ftkh_train_variant(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r, trv.size,
                                 _p(tri, _i32p), _p(trv, _f32p), nte, _p(tei, _i32p),
                                 _p(tev, _f32p), _ptrs(a), _ptrs(b), lr_a, lr_b, reg_a, reg_b,
                                 epochs, m, workers, int(store_c), seed & M64,
                                 _p(out["loss"], _f64p), _p(out["rmse"], _f64p),
                                 _p(out["mae"], _f64p), _p(out["seconds"], _f64p),
                                 _p(reads, _i64p), _p(mults, _i64p), buf, cap,
                                 VARIANTS[variant]))
    out["reads"], out["mults"] = reads, mults
    out["jsonl"] = buf.value.decode()
    return out


def loss(dims, ranks, r, idx, vals, a, b, reg_a, reg_b, workers=1):
    dims, ranks, idx = _i32(dims), _i32(ranks), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    v = C.c_double()
    _ck(lib().ftkh_loss(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r, vals.size,
                        _p(idx, _i32p), _p(vals, _f32p), _ptrs(a), _ptrs(b), reg_a, reg_b,
                        workers, C.byref(v)))
    return v.value


def evaluate(dims, ranks, r, idx, vals, a, b, workers=1):
    dims, ranks, idx = _i32(dims), _i32(ranks), _i32(idx)
    vals = np.ascontiguousarray(vals, np.float32)
    rm, ma = C.c_double(), C.c_double()
    _ck(lib().ftkh_evaluate(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r, vals.size,
                            _p(idx, _i32p), _p(vals, _f32p), _ptrs(a), _ptrs(b), workers,
                            C.byref(rm), C.byref(ma)))
    return rm.value, ma.value


def predicted_costs(order, m, r, ranks):
    ranks = _i32(ranks)
    out = np.zeros(4, np.int64)
    _ck(lib().ftkh_predicted_costs(order, m, r, _p(ranks, _i32p), _p(out, _i64p)))
    return out
