"""Storage scheme (EpochOptions.store_c) on the GPU: the core
phase reads C rows from the C cache (CCache::build/refresh, decomposition.cpp
:74-107; stage_c_rows_from_cache :299-314) instead of computing A B.

* deterministic mode: bit-exact against the reference's store_c epoch
  (golden fixtures) through the C-ABI and through ftk::epoch_plus;
* Hogwild mode: the core gradient (order-independent sum) against the
  oracle's storage-scheme sum, on the warp-specialised sweep (N = 3,
  J = R = 32) and on the CUDA-core sweep (other shapes).
"""
import numpy as np
import pytest

import oracle as O
import paper_2404_10087_b200 as eng
from golden_io import bits_equal, load, model, names, tensor
import datagen as synth
from paper_2404_10087_b200 import host

pytestmark = pytest.mark.gpu
DET, HOG = eng.MODE_DETERMINISTIC, eng.MODE_HOGWILD


@pytest.mark.parametrize("name", names("storec_"))
def test_storage_scheme_deterministic_bit_exact(session, name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    cap = int(z["cap"])
    session.upload_tensor(0, t.dims, t.idx, t.vals)
    session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
    session.set_option("store_c", 1)
    try:
        session.factor_phase(0, z["plan1"], cap, lr_a, reg_a, DET)
        session.core_phase(0, z["plan2"], cap, lr_b, reg_b, DET)
    finally:
        session.set_option("store_c", 0)
    a, b = session.download_model()
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(a[n], want.a[n]), f"A{n}"
        assert bits_equal(b[n], want.b[n]), f"B{n}"


def test_storage_scheme_cxx_api_epoch_plus():
    z = load("storec_j16")
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    host.set_device_options(mode=0, precision=0, exact_eval=True)
    a, b = [x.copy() for x in m.a], [x.copy() for x in m.b]
    host.epoch_plus(t.dims, m.ranks, m.r, t.idx, t.vals, a, b, int(z["seed"]), lr_a, lr_b,
                    reg_a, reg_b, int(z["cap"]), workers=1, store_c=True)
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(a[n], want.a[n]) and bits_equal(b[n], want.b[n])


@pytest.mark.parametrize("prec", [eng.PREC_FP32, eng.PREC_TF32])
@pytest.mark.parametrize("shape", [(3, 32, 32), (3, 16, 16), (4, 8, 8)], ids=str)
def test_storage_scheme_hogwild_core_gradient(session, shape, prec):
    order, j, r = shape
    dims = (300, 200, 100, 90)[:order]
    c, _, _ = synth.planted_numpy(dims, 40000, 3, j, r, 0.05)
    t = O.Tensor(c.dims, c.idx, c.vals)
    scale = host.default_init_scale(float(np.mean(np.abs(t.vals))), order, r, [j] * order)
    a, b = host.init_model(t.dims, [j] * order, r, 9, scale)
    m = O.Model(t.dims, np.array([j] * order, np.int32), r, a, b)
    session.upload_tensor(0, t.dims, t.idx, t.vals)
    session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
    session.set_option("precision", prec)
    session.set_option("store_c", 1)
    try:
        _, g = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
    finally:
        session.set_option("store_c", 0)
        session.set_option("precision", eng.PREC_FP32)
    want = O.COracle.core_phase(t, m.copy(), host.global_plan(t.nnz, 16, 1), 16, 1e-3, 1e-4,
                                store_c=True)
    # fp32: reassociation only; tf32: the G GEMM's operands (C itself is exact)
    tol = 2e-5 if prec == eng.PREC_FP32 else 1e-2
    np.testing.assert_allclose(g, want, rtol=tol, atol=tol * np.abs(want).max())
