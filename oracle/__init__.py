"""TEST INFRASTRUCTURE ONLY: CPU oracles for the FastTuckerPlus hot path.

Two oracles live here, both loaded through ctypes:

* ``C``   -- ``oracle/build/libftk_oracle.so``, the plain-C restatement of the
  reference algorithm (``oracle/ftk_oracle.c``).  Always buildable.
* ``REF`` -- ``oracle/_ref/libftkref.so``, the unmodified reference library
  (``/root/reference/proj/src``) compiled with its own Release flags plus the
  ``oracle/ref_capi.cpp`` shim.  Present when it was built in the container
  (it travels to the GPU box with the snapshot); ``None`` otherwise.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this package.  The engine (``paper_2404_10087_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_C_PATH = os.path.join(HERE, "build", "libftk_oracle.so")
_REF_PATH = os.path.join(HERE, "_ref", "libftkref.so")

_f32p = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_fpp = C.POINTER(_f32p)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _ptr_array(arrs):
    out = (_f32p * len(arrs))()
    for i, a in enumerate(arrs):
        assert a.dtype == np.float32 and a.flags.c_contiguous
        out[i] = a.ctypes.data_as(_f32p)
    return out


# ---------------------------------------------------------------------------
# Host-side problem containers (numpy), shared by tests / bench legs.


@dataclass
class Tensor:
    """COO tensor, AoS indices [nnz, order] int32 (0-based), fp32 values."""

    dims: np.ndarray
    idx: np.ndarray
    vals: np.ndarray

    @property
    def order(self) -> int:
        return int(self.dims.shape[0])

    @property
    def nnz(self) -> int:
        return int(self.vals.shape[0])


@dataclass
class Model:
    dims: np.ndarray
    ranks: np.ndarray
    r: int
    a: list = field(default_factory=list)
    b: list = field(default_factory=list)

    @property
    def order(self) -> int:
        return int(self.dims.shape[0])

    def copy(self) -> "Model":
        return Model(self.dims.copy(), self.ranks.copy(), self.r,
                     [x.copy() for x in self.a], [x.copy() for x in self.b])


def random_tensor(dims, nnz, seed, lo=0.0, hi=1.0) -> Tensor:
    """Distinct uniform tuples, uniform values (numpy; not the reference RNG)."""
    rng = np.random.default_rng(seed)
    dims = np.asarray(dims, dtype=np.int64)
    cells = int(np.prod(dims.astype(np.float64)))
    assert nnz <= cells
    keys = np.empty(0, dtype=np.int64)
    while keys.size < nnz:
        need = nnz - keys.size
        cols = [rng.integers(0, d, size=need + need // 8 + 16) for d in dims]
        k = np.zeros_like(cols[0])
        for c, d in zip(cols, dims):
            k = k * d + c
        keys = np.unique(np.concatenate([keys, k]))
    keys = rng.permutation(keys)[:nnz]
    idx = np.empty((nnz, dims.size), dtype=np.int32)
    rem = keys.copy()
    for n in range(dims.size - 1, -1, -1):
        idx[:, n] = rem % dims[n]
        rem //= dims[n]
    vals = rng.uniform(lo, hi, size=nnz).astype(np.float32)
    return Tensor(dims.astype(np.int32), idx, vals)


def random_model(dims, ranks, r, seed, scale=0.5) -> Model:
    rng = np.random.default_rng(seed)
    dims = np.asarray(dims, dtype=np.int32)
    ranks = np.asarray(ranks, dtype=np.int32)
    a = [rng.uniform(0, scale, size=(int(d), int(j))).astype(np.float32)
         for d, j in zip(dims, ranks)]
    b = [rng.uniform(0, scale, size=(int(j), r)).astype(np.float32) for j in ranks]
    return Model(dims, ranks, int(r), a, b)


# ---------------------------------------------------------------------------
# The plain-C restatement.


class _COracle:
    def __init__(self, path=_C_PATH):
        self.lib = L = C.CDLL(path)
        L.fo_batch_probe.argtypes = [C.c_int, _i32p, C.c_int, _fpp, _fpp, _i32p, _f32p,
                                     _i64p, C.c_int, C.c_int, C.c_float, C.c_float] + [_f32p] * 9
        L.fo_factor_phase.argtypes = [C.c_int, _i32p, C.c_int, _fpp, _fpp, C.c_int64, _i32p,
                                      _f32p, _i64p, C.c_int, C.c_float, C.c_float]
        L.fo_core_phase.argtypes = [C.c_int, _i32p, C.c_int, _fpp, _fpp, C.c_int64, _i32p,
                                    _f32p, _i64p, C.c_int, C.c_float, C.c_float, _f32p, C.c_int]
        L.fo_fasttucker_factor_block.argtypes = [C.c_int, _i32p, C.c_int, _fpp, _fpp, _i32p,
                                                 _f32p, _i64p, _i64p, C.c_int64, C.c_int,
                                                 C.c_int, C.c_float, C.c_float]
        L.fo_fasttucker_core_block.argtypes = [C.c_int, _i32p, C.c_int, _fpp, _fpp, C.c_int64,
                                               _i32p, _f32p, _i64p, C.c_int, C.c_int, C.c_float,
                                               C.c_float]
        L.fo_ccache_refresh.argtypes = [C.c_int32, C.c_int, C.c_int, _f32p, _f32p, _f32p]
        for fn in ("fo_fastertucker_factor_block", "fo_fastertucker_core_block"):
            getattr(L, fn).argtypes = [C.c_int, _i32p, _i32p, C.c_int, _fpp, _fpp, _fpp, _i32p,
                                       _f32p, _i64p, _i64p, C.c_int64, C.c_int, C.c_float,
                                       C.c_float]
        L.fo_predict.argtypes = [C.c_int, _i32p, C.c_int, _fpp, _fpp, _i32p]
        L.fo_predict.restype = C.c_double
        L.fo_loss.argtypes = [C.c_int, _i32p, _i32p, C.c_int, _fpp, _fpp, C.c_int64, _i32p,
                              _f32p, C.c_double, C.c_double, C.c_int]
        L.fo_loss.restype = C.c_double
        L.fo_evaluate.argtypes = [C.c_int, _i32p, C.c_int, _fpp, _fpp, C.c_int64, _i32p, _f32p,
                                  C.c_int, _f64p, _f64p]
        L.fo_predicted_costs.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i64p]

    def batch_probe(self, t: Tensor, m: Model, rows, cap, lr_a, reg_a):
        """Runs one batch; mutates m.a like update_factors_plus. Returns dict."""
        return _probe(self.lib.fo_batch_probe, t, m, rows, cap, lr_a, reg_a, c_oracle=True)

    def factor_phase(self, t: Tensor, m: Model, perm, cap, lr_a, reg_a):
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        rc = self.lib.fo_factor_phase(m.order, _p(m.ranks, _i32p), m.r, _ptr_array(m.a),
                                      _ptr_array(m.b), t.nnz, _p(t.idx, _i32p),
                                      _p(t.vals, _f32p), _p(perm, _i64p), cap, lr_a, reg_a)
        assert rc == 0

    def fasttucker_factor_block(self, t: Tensor, m: Model, perm, boff, cap, mode, lr_a, reg_a):
        """FastTucker factor block of `mode` over a per-bucket plan (in place)."""
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        boff = np.ascontiguousarray(boff, dtype=np.int64)
        rc = self.lib.fo_fasttucker_factor_block(
            m.order, _p(m.ranks, _i32p), m.r, _ptr_array(m.a), _ptr_array(m.b),
            _p(t.idx, _i32p), _p(t.vals, _f32p), _p(perm, _i64p), _p(boff, _i64p),
            boff.size - 1, cap, mode, lr_a, reg_a)
        assert rc == 0

    def fasttucker_core_block(self, t: Tensor, m: Model, perm, cap, mode, lr_b, reg_b):
        """FastTucker core block of `mode` over a global plan (in place)."""
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        rc = self.lib.fo_fasttucker_core_block(
            m.order, _p(m.ranks, _i32p), m.r, _ptr_array(m.a), _ptr_array(m.b), t.nnz,
            _p(t.idx, _i32p), _p(t.vals, _f32p), _p(perm, _i64p), cap, mode, lr_b, reg_b)
        assert rc == 0

    def ccache_build(self, m: Model):
        """CCache::build (decomposition.cpp:84-87): C_n = A_n B_n for every mode."""
        out = []
        for n in range(m.order):
            c = np.zeros((int(m.dims[n]), m.r), np.float32)
            self.lib.fo_ccache_refresh(int(m.dims[n]), int(m.ranks[n]), m.r,
                                       _p(np.ascontiguousarray(m.a[n]), _f32p),
                                       _p(np.ascontiguousarray(m.b[n]), _f32p), _p(c, _f32p))
            out.append(c)
        return out

    def fastertucker_block(self, factor, t: Tensor, m: Model, cache, perm, batch_off, mode, lr,
                           reg):
        """FasterTucker factor (factor=True) or core block of `mode` over a
        complement-keyed per-bucket plan cut into batches (in place; the
        mode's cache rows are refreshed at the end)."""
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        bo = np.ascontiguousarray(batch_off, dtype=np.int64)
        fn = self.lib.fo_fastertucker_factor_block if factor else self.lib.fo_fastertucker_core_block
        rc = fn(m.order, _p(m.dims, _i32p), _p(m.ranks, _i32p), m.r, _ptr_array(m.a),
                _ptr_array(m.b), _ptr_array(cache), _p(t.idx, _i32p), _p(t.vals, _f32p),
                _p(perm, _i64p), _p(bo, _i64p), bo.size - 1, mode, lr, reg)
        assert rc == 0

    def core_phase(self, t: Tensor, m: Model, perm, cap, lr_b, reg_b, store_c=False):
        """store_c: storage scheme (C rows from the C cache, decomposition.cpp:668-691)."""
        perm = np.ascontiguousarray(perm, dtype=np.int64)
        g = np.zeros(int(np.sum(m.ranks)) * m.r, dtype=np.float32)
        rc = self.lib.fo_core_phase(m.order, _p(m.ranks, _i32p), m.r, _ptr_array(m.a),
                                    _ptr_array(m.b), t.nnz, _p(t.idx, _i32p),
                                    _p(t.vals, _f32p), _p(perm, _i64p), cap, lr_b, reg_b,
                                    _p(g, _f32p), int(store_c))
        if rc != 0:
            raise RuntimeError("apply_core_update: empty tensor")
        return g

    def predict(self, m: Model, idx):
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        return self.lib.fo_predict(m.order, _p(m.ranks, _i32p), m.r, _ptr_array(m.a),
                                   _ptr_array(m.b), _p(idx, _i32p))

    def loss(self, m: Model, t: Tensor, reg_a, reg_b, workers=1):
        return self.lib.fo_loss(m.order, _p(m.dims, _i32p), _p(m.ranks, _i32p), m.r,
                                _ptr_array(m.a), _ptr_array(m.b), t.nnz, _p(t.idx, _i32p),
                                _p(t.vals, _f32p), reg_a, reg_b, workers)

    def evaluate(self, m: Model, t: Tensor, workers=1):
        rm, ma = C.c_double(), C.c_double()
        self.lib.fo_evaluate(m.order, _p(m.ranks, _i32p), m.r, _ptr_array(m.a),
                             _ptr_array(m.b), t.nnz, _p(t.idx, _i32p), _p(t.vals, _f32p),
                             workers, C.byref(rm), C.byref(ma))
        return rm.value, ma.value

    def predicted_costs(self, order, m, r, ranks):
        ranks = np.ascontiguousarray(ranks, dtype=np.int32)
        out = np.zeros(4, dtype=np.int64)
        self.lib.fo_predicted_costs(order, m, r, _p(ranks, _i32p), _p(out, _i64p))
        return out


def _probe(fn, t, m, rows, cap, lr_a, reg_a, c_oracle, handles=None):
    order, r = m.order, m.r
    jmax = int(np.max(m.ranks))
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    out = dict(
        c=np.zeros((order, cap, r), np.float32), d=np.zeros((order, cap, r), np.float32),
        u=np.zeros((order, cap, jmax), np.float32), xhat_f=np.zeros(cap, np.float32),
        resid_f=np.zeros(cap, np.float32), xhat_c=np.zeros(cap, np.float32),
        resid_c=np.zeros(cap, np.float32), a_new=np.zeros((order, cap, jmax), np.float32),
        g=np.zeros((order, jmax, r), np.float32))
    tail = [_p(out[k], _f32p) for k in ("c", "d", "u", "xhat_f", "resid_f", "xhat_c",
                                         "resid_c", "a_new", "g")]
    if c_oracle:
        rc = fn(order, _p(m.ranks, _i32p), r, _ptr_array(m.a), _ptr_array(m.b),
                _p(t.idx, _i32p), _p(t.vals, _f32p), _p(rows, _i64p), rows.size, cap,
                lr_a, reg_a, *tail)
    else:
        th, mh = handles
        rc = fn(th, mh, _p(rows, _i64p), rows.size, cap, lr_a, reg_a, *tail)
    assert rc == 0
    return out


# ---------------------------------------------------------------------------
# The reference library itself.


class _Ref:
    def __init__(self, path=_REF_PATH):
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_tensor_new.restype = C.c_void_p
        L.ref_tensor_new.argtypes = [C.c_int, _i32p, C.c_int64, _i32p, _f32p]
        L.ref_tensor_nnz.restype = C.c_int64
        L.ref_tensor_nnz.argtypes = [C.c_void_p]
        L.ref_tensor_get.argtypes = [C.c_void_p, _i32p, _i32p, _f32p]
        L.ref_tensor_free.argtypes = [C.c_void_p]
        L.ref_tensor_validate.argtypes = [C.c_void_p]
        L.ref_split.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.POINTER(C.c_void_p),
                                C.POINTER(C.c_void_p)]
        L.ref_load_coo.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_global_plan.argtypes = [C.c_int64, C.c_int, C.c_uint64, _i64p]
        L.ref_model_new.restype = C.c_void_p
        L.ref_model_new.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, _fpp, _fpp]
        L.ref_model_init.argtypes = [C.c_int, _i32p, _i32p, C.c_int32, C.c_uint64, C.c_float,
                                     C.POINTER(C.c_void_p)]
        L.ref_model_get.argtypes = [C.c_void_p, _fpp, _fpp]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_int]
        L.ref_default_init_scale.restype = C.c_float
        L.ref_default_init_scale.argtypes = [C.c_double, C.c_int, C.c_int32, _i32p]
        L.ref_predict.restype = C.c_double
        L.ref_predict.argtypes = [C.c_void_p, _i32p]
        L.ref_epoch_plus.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_float, C.c_float,
                                     C.c_float, C.c_int, C.c_int, C.c_int, C.c_uint64, _f64p,
                                     _i64p]
        L.ref_train.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_float,
                                C.c_float, C.c_float, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_uint64, _f64p, _f64p, _f64p, _f64p, _i64p, _i64p]
        L.ref_train_variant.argtypes = list(L.ref_train.argtypes) + [C.c_int]
        L.ref_loss.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int, _f64p]
        L.ref_evaluate.argtypes = [C.c_void_p, C.c_void_p, C.c_int, _f64p, _f64p]
        L.ref_batch_probe.argtypes = [C.c_void_p, C.c_void_p, _i64p, C.c_int, C.c_int, C.c_float,
                                      C.c_float] + [_f32p] * 9
        L.ref_predicted_costs.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i64p]
        L.ref_epoch_fastertucker.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_float,
                                             C.c_float, C.c_float, C.c_int, C.c_int, C.c_int,
                                             C.c_uint64, _i64p]
        L.ref_per_bucket_plan.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                          _i64p, _i64p, _i64p]
        L.ref_epoch_fasttucker.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_float,
                                           C.c_float, C.c_float, C.c_int, C.c_int, C.c_int,
                                           C.c_uint64, _f64p, _i64p]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())

    # -- handles
    def tensor(self, t: Tensor):
        return self.lib.ref_tensor_new(t.order, _p(t.dims, _i32p), t.nnz, _p(t.idx, _i32p),
                                       _p(t.vals, _f32p))

    def tensor_to_np(self, h, order) -> Tensor:
        nnz = self.lib.ref_tensor_nnz(h)
        dims = np.zeros(order, np.int32)
        idx = np.zeros((nnz, order), np.int32)
        vals = np.zeros(nnz, np.float32)
        self.lib.ref_tensor_get(h, _p(dims, _i32p), _p(idx, _i32p), _p(vals, _f32p))
        return Tensor(dims, idx, vals)

    def model(self, m: Model):
        return self.lib.ref_model_new(m.order, _p(m.dims, _i32p), _p(m.ranks, _i32p), m.r,
                                      _ptr_array(m.a), _ptr_array(m.b))

    def model_to_np(self, h, like: Model) -> Model:
        out = like.copy()
        self.lib.ref_model_get(h, _ptr_array(out.a), _ptr_array(out.b))
        return out

    def free_tensor(self, h):
        self.lib.ref_tensor_free(h)

    def free_model(self, h):
        self.lib.ref_model_free(h)

    # -- API
    def init_model(self, dims, ranks, r, seed, scale) -> Model:
        dims = np.ascontiguousarray(dims, np.int32)
        ranks = np.ascontiguousarray(ranks, np.int32)
        h = C.c_void_p()
        self._check(self.lib.ref_model_init(dims.size, _p(dims, _i32p), _p(ranks, _i32p), r,
                                            seed, scale, C.byref(h)))
        like = Model(dims, ranks, int(r),
                     [np.zeros((int(d), int(j)), np.float32) for d, j in zip(dims, ranks)],
                     [np.zeros((int(j), int(r)), np.float32) for j in ranks])
        out = self.model_to_np(h, like)
        self.free_model(h)
        return out

    def derive_seed(self, base, path) -> int:
        """ftkref::derive_seed (common.hpp:43-48)."""
        arr = (C.c_uint64 * len(path))(*[int(x) & (2**64 - 1) for x in path])
        return int(self.lib.ref_derive_seed(int(base) & (2**64 - 1), arr, len(path)))

    def default_init_scale(self, mean_abs, order, r, ranks):
        ranks = np.ascontiguousarray(ranks, np.int32)
        return self.lib.ref_default_init_scale(mean_abs, order, r, _p(ranks, _i32p))

    def global_plan(self, nnz, m, seed):
        out = np.zeros(nnz, np.int64)
        self._check(self.lib.ref_global_plan(nnz, m, seed, _p(out, _i64p)))
        return out

    def split(self, t: Tensor, frac, seed):
        h = self.tensor(t)
        tr, te = C.c_void_p(), C.c_void_p()
        try:
            self._check(self.lib.ref_split(h, frac, seed, C.byref(tr), C.byref(te)))
            out = self.tensor_to_np(tr, t.order), self.tensor_to_np(te, t.order)
            self.free_tensor(tr)
            self.free_tensor(te)
            return out
        finally:
            self.free_tensor(h)

    def predict(self, m: Model, idx):
        mh = self.model(m)
        idx = np.ascontiguousarray(idx, np.int32)
        v = self.lib.ref_predict(mh, _p(idx, _i32p))
        self.free_model(mh)
        return v

    def epoch_plus(self, t: Tensor, m: Model, seed, lr_a=1e-3, lr_b=1e-3, reg_a=1e-4,
                   reg_b=1e-4, batch=16, workers=1, store_c=False):
        """Runs ftkref::epoch_plus; returns (new model, seconds[2], counters[10])."""
        th, mh = self.tensor(t), self.model(m)
        secs = np.zeros(2, np.float64)
        cnt = np.zeros(10, np.int64)
        try:
            self._check(self.lib.ref_epoch_plus(th, mh, lr_a, lr_b, reg_a, reg_b, batch,
                                                workers, int(store_c), seed, _p(secs, _f64p),
                                                _p(cnt, _i64p)))
            return self.model_to_np(mh, m), secs, cnt
        finally:
            self.free_tensor(th)
            self.free_model(mh)

    def timed_epochs(self, t: Tensor, m: Model, seeds, lr_a=1e-3, lr_b=1e-3, reg_a=1e-4,
                     reg_b=1e-4, batch=16, workers=1):
        """ftkref::epoch_plus once per seed on ONE tensor/model handle (no
        per-epoch copies); returns (final model, [[factor s, core s], ...])."""
        th, mh = self.tensor(t), self.model(m)
        out = []
        try:
            for seed in seeds:
                secs = np.zeros(2, np.float64)
                self._check(self.lib.ref_epoch_plus(th, mh, lr_a, lr_b, reg_a, reg_b, batch,
                                                    workers, 0, seed, _p(secs, _f64p), None))
                out.append([float(secs[0]), float(secs[1])])
            return self.model_to_np(mh, m), out
        finally:
            self.free_tensor(th)
            self.free_model(mh)

    def per_bucket_plan(self, t: Tensor, mode, m, seed, keying=0):
        """EpochPlan::per_bucket positions and bucket offsets (plan order)."""
        th = self.tensor(t)
        perm = np.zeros(t.nnz, np.int64)
        boff = np.zeros(t.nnz + 2, np.int64)
        nb = np.zeros(1, np.int64)
        try:
            self._check(self.lib.ref_per_bucket_plan(th, mode, keying, m, seed, _p(perm, _i64p),
                                                     _p(boff, _i64p), _p(nb, _i64p)))
            return perm, boff[: int(nb[0]) + 1].copy()
        finally:
            self.free_tensor(th)

    def epoch_fasttucker(self, t: Tensor, m: Model, seed, lr_a=1e-3, lr_b=1e-3, reg_a=1e-4,
                         reg_b=1e-4, batch=16, workers=1, canonical=False):
        """Runs ftkref::epoch_fasttucker (fixed-mode indices); returns (new model,
        counters[10])."""
        th, mh = self.tensor(t), self.model(m)
        secs = np.zeros(2, np.float64)
        cnt = np.zeros(10, np.int64)
        try:
            self._check(self.lib.ref_epoch_fasttucker(th, mh, lr_a, lr_b, reg_a, reg_b, batch,
                                                      workers, int(canonical), seed,
                                                      _p(secs, _f64p), _p(cnt, _i64p)))
            return self.model_to_np(mh, m), cnt
        finally:
            self.free_tensor(th)
            self.free_model(mh)

    def epoch_fastertucker(self, t: Tensor, m: Model, seed, lr_a=1e-3, lr_b=1e-3, reg_a=1e-4,
                           reg_b=1e-4, batch=16, workers=1, canonical=False):
        """Runs ftkref::epoch_fastertucker (complement indices, fresh C cache);
        returns (new model, counters[10])."""
        th, mh = self.tensor(t), self.model(m)
        cnt = np.zeros(10, np.int64)
        try:
            self._check(self.lib.ref_epoch_fastertucker(th, mh, lr_a, lr_b, reg_a, reg_b, batch,
                                                        workers, int(canonical), seed,
                                                        _p(cnt, _i64p)))
            return self.model_to_np(mh, m), cnt
        finally:
            self.free_tensor(th)
            self.free_model(mh)

    def train(self, train: Tensor, test, m: Model, epochs, seed, lr_a=1e-3, lr_b=1e-3,
              reg_a=1e-4, reg_b=1e-4, batch=16, workers=1, store_c=False, variant=0):
        """ftkref::train; variant 0 plus, 1 fasttucker, 2 fastertucker."""
        th = self.tensor(train)
        teh = self.tensor(test) if test is not None else None
        mh = self.model(m)
        out = {k: np.zeros(epochs, np.float64) for k in ("loss", "rmse", "mae", "seconds")}
        reads = np.zeros(epochs, np.int64)
        mults = np.zeros(epochs, np.int64)
        try:
            self._check(self.lib.ref_train_variant(
                th, teh, mh, lr_a, lr_b, reg_a, reg_b, epochs, batch, workers, int(store_c),
                seed, _p(out["loss"], _f64p), _p(out["rmse"], _f64p), _p(out["mae"], _f64p),
                _p(out["seconds"], _f64p), _p(reads, _i64p), _p(mults, _i64p), int(variant)))
            out["reads"], out["mults"] = reads, mults
            out["model"] = self.model_to_np(mh, m)
            return out
        finally:
            self.free_tensor(th)
            if teh is not None:
                self.free_tensor(teh)
            self.free_model(mh)

    def loss(self, m: Model, t: Tensor, reg_a, reg_b, workers=1):
        th, mh = self.tensor(t), self.model(m)
        v = C.c_double()
        try:
            self._check(self.lib.ref_loss(mh, th, reg_a, reg_b, workers, C.byref(v)))
            return v.value
        finally:
            self.free_tensor(th)
            self.free_model(mh)

    def evaluate(self, m: Model, t: Tensor, workers=1):
        th, mh = self.tensor(t), self.model(m)
        rm, ma = C.c_double(), C.c_double()
        try:
            self._check(self.lib.ref_evaluate(mh, th, workers, C.byref(rm), C.byref(ma)))
            return rm.value, ma.value
        finally:
            self.free_tensor(th)
            self.free_model(mh)

    def batch_probe(self, t: Tensor, m: Model, rows, cap, lr_a, reg_a):
        th, mh = self.tensor(t), self.model(m)
        try:
            out = _probe(self.lib.ref_batch_probe, t, m, rows, cap, lr_a, reg_a,
                         c_oracle=False, handles=(th, mh))
            newm = self.model_to_np(mh, m)
            for n in range(m.order):
                m.a[n][...] = newm.a[n]
            return out
        finally:
            self.free_tensor(th)
            self.free_model(mh)

    def predicted_costs(self, order, m, r, ranks):
        ranks = np.ascontiguousarray(ranks, dtype=np.int32)
        out = np.zeros(4, dtype=np.int64)
        self.lib.ref_predicted_costs(order, m, r, _p(ranks, _i32p), _p(out, _i64p))
        return out


def _load(cls, path):
    if not os.path.exists(path):
        return None
    return cls(path)


COracle = _load(_COracle, _C_PATH)
REF = _load(_Ref, _REF_PATH)
