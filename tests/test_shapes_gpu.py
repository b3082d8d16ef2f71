"""Hogwild sweeps across every shape the BASELINE configs name (SURVEY.md §8
legend): order 3..6 (C4), J = R in {8, 16, 32, 64, 128} (C5 rank sweep) and
mixed J != R, for each precision.  Each kernel family the engine dispatches
to (warp-specialised tcgen05, synchronous tcgen05, fp32 CUDA cores) is
checked against the C oracle through two order-independent properties:

* the core sweep's gradient (a sum over all nonzeros of a read-only model)
  against the oracle's sequential fp32 sum;
* the factor sweep on a tensor whose nonzeros share no row in any mode, so
  Hogwild has no conflicts and every row's step must match the oracle's.
"""
import numpy as np
import pytest

import oracle as O
import paper_2404_10087_b200 as eng
import datagen as synth
from paper_2404_10087_b200 import host

pytestmark = pytest.mark.gpu
HOG = eng.MODE_HOGWILD

# (order, J, R)
SHAPES = [(3, 8, 8), (3, 16, 16), (3, 32, 32), (3, 64, 64), (3, 128, 128), (3, 16, 32),
          (3, 32, 16), (4, 16, 16), (5, 16, 16), (6, 16, 16), (4, 8, 8), (4, 32, 32)]
PRECS = [eng.PREC_FP32, eng.PREC_TF32, eng.PREC_3XTF32]
GRAD_TOL = {eng.PREC_FP32: 2e-5, eng.PREC_3XTF32: 3e-3, eng.PREC_TF32: 1e-2}
STEP_TOL = {eng.PREC_FP32: 1e-4, eng.PREC_3XTF32: 2e-2, eng.PREC_TF32: 2e-2}


def _model(t, j, r, seed=9):
    scale = host.default_init_scale(float(np.mean(np.abs(t.vals))), t.order, r, [j] * t.order)
    a, b = host.init_model(t.dims, [j] * t.order, r, seed, scale)
    return O.Model(t.dims, np.array([j] * t.order, np.int32), r, a, b)


def _planted(order, j, r, nnz):
    dims = (300, 200, 100, 90, 80, 70)[:order]
    t, _, _ = synth.planted_numpy(dims, nnz, 3, j, r, 0.05)
    return O.Tensor(t.dims, t.idx, t.vals)


def _id(shape):
    return "N%d-J%d-R%d" % shape


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("shape", SHAPES, ids=_id)
def test_core_gradient_all_shapes(session, shape, prec):
    order, j, r = shape
    nnz = 40000 if j * r <= 1024 else 6000
    t = _planted(order, j, r, nnz)
    m = _model(t, j, r)
    session.set_option("precision", prec)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        _, g = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
    finally:
        session.set_option("precision", eng.PREC_FP32)
    mc = m.copy()
    want = O.COracle.core_phase(t, mc, host.global_plan(t.nnz, 16, 1), 16, 1e-3, 1e-4)
    tol = GRAD_TOL[prec]
    assert np.isfinite(g).all()
    np.testing.assert_allclose(g, want, rtol=tol, atol=tol * np.abs(want).max())
    _, b = session.download_model()
    for n in range(order):
        np.testing.assert_allclose(b[n], mc.b[n], rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("shape", SHAPES, ids=_id)
def test_factor_distinct_rows_all_shapes(session, shape, prec):
    order, j, r = shape
    n = 1000 if j * r <= 1024 else 300
    mult = (1, 7, 13, 17, 19, 23)[:order]
    idx = np.stack([(np.arange(n) * p) % n for p in mult], 1).astype(np.int32)
    vals = np.linspace(1, 5, n).astype(np.float32)
    t = O.Tensor(np.array([n] * order, np.int32), idx, vals)
    m = _model(t, j, r)
    session.set_option("precision", prec)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        session.factor_phase(0, None, 16, 1e-2, 1e-3, HOG, seed=3)
    finally:
        session.set_option("precision", eng.PREC_FP32)
    a, _ = session.download_model()
    mc = m.copy()
    O.COracle.factor_phase(t, mc, np.arange(n), 16, 1e-2, 1e-3)
    tol = STEP_TOL[prec]
    for k in range(order):
        got, want = a[k] - m.a[k], mc.a[k] - m.a[k]
        assert np.isfinite(got).all()
        np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())


@pytest.mark.parametrize("core16", [0, 1, 2])
def test_core_gradient_tf32_and_f16_operand_paths(session, core16):
    """N = 3, J = R = 32 (the headline shape) has two single-pass core sweeps:
    tf32 rows copied into TMEM (core16 = 0) and one fp16 row tile read by both
    GEMMs (core16 = 1, the default).  Both must match the oracle."""
    t = _planted(3, 32, 32, 40000)
    m = _model(t, 32, 32)
    session.set_option("precision", eng.PREC_TF32)
    session.set_option("core16", core16)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        _, g = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
    finally:
        session.set_option("core16", 2)  # the default
        session.set_option("precision", eng.PREC_FP32)
    want = O.COracle.core_phase(t, m.copy(), host.global_plan(t.nnz, 16, 1), 16, 1e-3, 1e-4)
    tol = GRAD_TOL[eng.PREC_TF32]
    np.testing.assert_allclose(g, want, rtol=tol, atol=tol * np.abs(want).max())


@pytest.mark.parametrize("warps", [8, 16])
def test_factor_steps_8_and_16_epilogue_warps(session, warps):
    """N = 3, J = R = 32 has two factor sweeps: 8 epilogue warps (tc_ws) and
    16 (tc_wsg, 8 columns per warp).  Distinct rows: every step must match."""
    n = 1000
    idx = np.stack([(np.arange(n) * p) % n for p in (1, 7, 13)], 1).astype(np.int32)
    vals = np.linspace(1, 5, n).astype(np.float32)
    t = O.Tensor(np.array([n] * 3, np.int32), idx, vals)
    m = _model(t, 32, 32)
    session.set_option("precision", eng.PREC_TF32)
    session.set_option("factor_warps", warps)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        session.factor_phase(0, None, 16, 1e-2, 1e-3, HOG, seed=3)
    finally:
        session.set_option("factor_warps", 8)
        session.set_option("precision", eng.PREC_FP32)
    a, _ = session.download_model()
    mc = m.copy()
    O.COracle.factor_phase(t, mc, np.arange(n), 16, 1e-2, 1e-3)
    tol = STEP_TOL[eng.PREC_TF32]
    for k in range(3):
        got, want = a[k] - m.a[k], mc.a[k] - m.a[k]
        np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())


MULTI = [(3, 32, 32), (3, 64, 64), (3, 128, 128), (4, 16, 16)]


@pytest.mark.parametrize("shape", MULTI, ids=_id)
def test_core_gradient_many_tiles_per_cta(session, shape):
    """Enough nonzeros that every persistent CTA runs several tiles (> 2 x 148
    tiles of 128): the pipelines' stage reuse across tiles (C of tile k while
    G of tile k - 1 still holds its stage) is exercised, not just one pass."""
    order, j, r = shape
    t = _planted(order, j, r, 148 * 128 * 3 + 77)
    m = _model(t, j, r)
    session.set_option("precision", eng.PREC_TF32)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        _, g = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
    finally:
        session.set_option("precision", eng.PREC_FP32)
    want = O.COracle.core_phase(t, m.copy(), host.global_plan(t.nnz, 16, 1), 16, 1e-3, 1e-4)
    tol = GRAD_TOL[eng.PREC_TF32]
    assert np.isfinite(g).all()
    np.testing.assert_allclose(g, want, rtol=tol, atol=tol * np.abs(want).max())


@pytest.mark.parametrize("shape", MULTI, ids=_id)
def test_factor_distinct_rows_many_tiles_per_cta(session, shape):
    order, j, r = shape
    n = 148 * 128 * 2 + 51
    mult = (1, 7, 13, 17)[:order]
    idx = np.stack([(np.arange(n) * p) % n for p in mult], 1).astype(np.int32)
    vals = np.linspace(1, 5, n).astype(np.float32)
    t = O.Tensor(np.array([n] * order, np.int32), idx, vals)
    m = _model(t, j, r)
    session.set_option("precision", eng.PREC_TF32)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        session.factor_phase(0, None, 16, 1e-2, 1e-3, HOG, seed=3)
    finally:
        session.set_option("precision", eng.PREC_FP32)
    a, _ = session.download_model()
    mc = m.copy()
    O.COracle.factor_phase(t, mc, np.arange(n), 16, 1e-2, 1e-3)
    tol = STEP_TOL[eng.PREC_TF32]
    for k in range(order):
        got, want = a[k] - m.a[k], mc.a[k] - m.a[k]
        assert np.isfinite(got).all()
        np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())
