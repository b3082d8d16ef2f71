"""GPU parity: the B200 engine against the CPU oracle and the reference's
golden fixtures.  Deterministic mode is compared BIT-FOR-BIT (it reproduces
the reference's fp32 rounding sequence); Hogwild mode, whose update order
differs by design, is compared through order-independent properties and
the RMSE tolerance of BASELINE.json (1e-3).

All calls go through the C-ABI (libftkcu.so) or the ftk:: C++ API
(libftk.so) -- the same libraries a C++ caller links.
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


def upload(s, t, m, slot=0):
    s.upload_tensor(slot, t.dims, t.idx, t.vals)
    s.upload_model(m.dims, m.ranks, m.r, m.a, m.b)


# ---------------------------------------------------------------------------
# per-batch pipeline (reference decomposition.hpp:86-124)


@pytest.mark.parametrize("name", names("probe_"))
def test_batch_probe_bit_exact_vs_golden(session, name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    upload(session, t, m)
    out = session.batch_probe(0, z["rows"], int(z["cap"]), float(z["lr_a"]), float(z["reg_a"]))
    for key, v in out.items():
        assert bits_equal(v, z[f"out_{key}"]), key
    a, _ = session.download_model()
    for n in range(m.order):
        assert bits_equal(a[n], z[f"after_a{n}"]), n


@pytest.mark.parametrize("case", range(8))
def test_batch_probe_bit_exact_vs_oracle_random_shapes(session, case):
    rng = np.random.default_rng(1000 + case)
    order = int(rng.integers(2, 7))
    dims = [int(x) for x in rng.integers(2, 9, size=order)]
    t = O.random_tensor(dims, int(min(np.prod(dims), 60)), case, -2.0, 4.0)
    ranks = [int(x) for x in rng.integers(1, 70, size=order)]
    r = int(rng.integers(1, 70))
    cap = int(rng.integers(1, 40))
    rows = rng.choice(t.nnz, size=int(rng.integers(1, cap + 1)), replace=True)
    m = O.random_model(dims, ranks, r, case, 0.8)
    m.b[0] -= 0.3  # negative entries exercise signed zeros
    mc = m.copy()
    want = O.COracle.batch_probe(t, mc, rows, cap, 0.03, 0.002)
    upload(session, t, m)
    got = session.batch_probe(0, rows, cap, 0.03, 0.002)
    for key in want:
        assert bits_equal(got[key], want[key]), key
    a, _ = session.download_model()
    for n in range(order):
        assert bits_equal(a[n], mc.a[n])


# ---------------------------------------------------------------------------
# deterministic epochs (reference decomposition.cpp:623-705, workers == 1)


@pytest.mark.parametrize("name", names("epoch_"))
def test_deterministic_epoch_bit_exact_vs_golden(session, name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    cap = int(z["cap"])
    upload(session, t, m)
    session.factor_phase(0, z["plan1"], cap, lr_a, reg_a, DET)
    session.core_phase(0, z["plan2"], cap, lr_b, reg_b, DET)
    a, b = session.download_model()
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(a[n], want.a[n]), f"A{n}"
        assert bits_equal(b[n], want.b[n]), f"B{n}"
    session.set_option("eval", eng.EVAL_EXACT)
    out = session.eval(0, 1, 1e-3, 2e-3)
    assert out[0] + out[2] == float(z["loss_w1"])
    out3 = session.eval(0, 3, 1e-3, 2e-3)
    assert out3[0] + out3[2] == float(z["loss_w3"])
    out4 = session.eval(0, 4, 0.0, 0.0)
    n = t.nnz
    assert (np.sqrt(out4[0] / n), out4[1] / n) == tuple(z["eval_w4"])


def test_cxx_api_epoch_plus_matches_golden_counters_and_model():
    z = load("epoch_cap5")
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    host.set_device_options(mode=0, precision=0, exact_eval=True)
    secs, cnt = host.epoch_plus(t.dims, m.ranks, m.r, t.idx, t.vals, m.a, m.b, int(z["seed"]),
                                lr_a, lr_b, reg_a, reg_b, m=int(z["cap"]), workers=1)
    want = model(z, "new_")
    for n in range(3):
        assert bits_equal(m.a[n], want.a[n]) and bits_equal(m.b[n], want.b[n])
    assert np.array_equal(cnt, z["counters"])
    assert secs[0] > 0 and secs[1] > 0


def test_cxx_api_train_matches_golden_trajectory():
    z = load("train_small")
    a = [z[f"m0_a{n}"].copy() for n in range(3)]
    b = [z[f"m0_b{n}"].copy() for n in range(3)]
    host.set_device_options(mode=0, precision=0, exact_eval=True)
    h = host.train(z["full_dims"], [8, 8, 8], 8, z["tr_idx"], z["tr_vals"], z["te_idx"],
                   z["te_vals"], a, b, epochs=4, seed=1, workers=1)
    assert np.array_equal(h["loss"], z["loss"])
    assert np.array_equal(h["rmse"], z["rmse"])
    assert np.array_equal(h["mae"], z["mae"])
    assert np.array_equal(h["reads"], z["reads"]) and np.array_equal(h["mults"], z["mults"])
    for n in range(3):
        assert bits_equal(a[n], z[f"final_a{n}"]) and bits_equal(b[n], z[f"final_b{n}"])
    lines = h["jsonl"].strip().split("\n")
    assert len(lines) == 4 and '"epoch":1' in lines[0]


def test_deterministic_edge_cases(session):
    # nnz < M, nnz == 1, M == 1 and a duplicate-heavy tiny tensor.
    for dims, nnz, cap in [([3, 3, 2], 18, 16), ([2, 2, 2], 1, 16), ([5, 4, 3], 40, 1),
                           ([4, 4, 4], 33, 64)]:
        t = O.random_tensor(dims, nnz, nnz, 0.0, 2.0)
        m = O.random_model(dims, [3, 5, 2], 4, nnz)
        p1 = host.global_plan(t.nnz, cap, 11)
        p2 = host.global_plan(t.nnz, cap, 12)
        upload(session, t, m)
        session.factor_phase(0, p1, cap, 0.05, 0.01, DET)
        session.core_phase(0, p2, cap, 0.05, 0.01, DET)
        a, b = session.download_model()
        O.COracle.factor_phase(t, m, p1, cap, 0.05, 0.01)
        O.COracle.core_phase(t, m, p2, cap, 0.05, 0.01)
        for n in range(3):
            assert bits_equal(a[n], m.a[n]) and bits_equal(b[n], m.b[n])


def test_empty_tensor_core_phase_raises(session):
    t = O.Tensor(np.array([3, 3, 3], np.int32), np.zeros((0, 3), np.int32),
                 np.zeros(0, np.float32))
    m = O.random_model([3, 3, 3], [2, 2, 2], 2, 1)
    upload(session, t, m)
    session.factor_phase(0, np.zeros(0, np.int64), 16, 1e-3, 1e-4, DET)
    with pytest.raises(eng.FtkError, match="empty tensor"):
        session.core_phase(0, np.zeros(0, np.int64), 16, 1e-3, 1e-4, DET)


def test_out_of_range_index_rejected(session):
    with pytest.raises(eng.FtkError, match="out of range"):
        session.upload_tensor(0, np.array([2, 2, 2], np.int32),
                              np.array([[0, 1, 2]], np.int32), np.array([1.0], np.float32))


def test_out_of_range_plan_rejected(session):
    t = O.random_tensor([6, 5, 4], 50, 3, 1.0, 5.0)
    m = O.random_model([6, 5, 4], [4, 4, 4], 4, 3)
    upload(session, t, m)
    bad = host.global_plan(t.nnz, 16, 5)
    bad[7] = t.nnz  # one past the end
    with pytest.raises(eng.FtkError, match="plan entry 7"):
        session.factor_phase(0, bad, 16, 1e-3, 1e-4, DET)
    bad[7] = -1
    with pytest.raises(eng.FtkError, match="plan entry 7"):
        session.core_phase(0, bad, 16, 1e-3, 1e-4, DET)


def test_cxx_api_sees_in_place_edits_of_a_cached_tensor():
    """The ftk:: layer caches tensors on the device; an in-place edit of one
    value anywhere (not just at sampled positions) must reach the device."""
    t = O.random_tensor([50, 40, 30], 5000, 4, 1.0, 5.0)
    m = O.random_model([50, 40, 30], [8, 8, 8], 8, 4)
    host.set_device_options(mode=0, precision=0, exact_eval=True)
    before = host.loss(t.dims, m.ranks, m.r, t.idx, t.vals, m.a, m.b, 0.0, 0.0)
    assert before == O.COracle.loss(m, t, 0.0, 0.0, 1)
    t.vals[4999 - 13] += 1.0  # not on the old 64-sample grid (step = nnz / 64)
    after = host.loss(t.dims, m.ranks, m.r, t.idx, t.vals, m.a, m.b, 0.0, 0.0)
    assert after == O.COracle.loss(m, t, 0.0, 0.0, 1) and after != before


@pytest.mark.parametrize("ranks,r", [([128, 128, 128], 128), ([16] * 6, 16), ([64, 32, 8], 48)])
def test_deterministic_large_ranks_and_order(session, ranks, r):
    order = len(ranks)
    dims = [30, 20, 10, 6, 5, 4][:order]
    t = O.random_tensor(dims, 400, 3, 1.0, 5.0)
    m = O.random_model(dims, ranks, r, 4, 2.0 / np.sqrt(max(ranks)) * (3.0 / r) ** (1 / (2 * order)))
    p1, p2 = host.global_plan(t.nnz, 16, 5), host.global_plan(t.nnz, 16, 6)
    upload(session, t, m)
    session.factor_phase(0, p1, 16, 1e-3, 1e-4, DET)
    session.core_phase(0, p2, 16, 1e-3, 1e-4, DET)
    a, b = session.download_model()
    O.COracle.factor_phase(t, m, p1, 16, 1e-3, 1e-4)
    O.COracle.core_phase(t, m, p2, 16, 1e-3, 1e-4)
    for n in range(order):
        assert bits_equal(a[n], m.a[n]) and bits_equal(b[n], m.b[n])


def test_c1_one_epoch_bit_exact(session):
    """Config 1 (10k x 10k x 1k, 1M nnz, J = R = 16): one full deterministic
    epoch at the reference's scale, bit-identical to the oracle."""
    cfg = synth.CONFIGS["c1"]
    c = synth.uniform_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], cfg["lo"], cfg["hi"])
    t = O.Tensor(c.dims, c.idx, c.vals)
    scale = host.default_init_scale(float(np.mean(np.abs(t.vals))), 3, 16, [16] * 3)
    a, b = host.init_model(t.dims, [16] * 3, 16, host.derive_seed(1, [77]), scale)
    m = O.Model(t.dims, np.array([16] * 3, np.int32), 16, a, b)
    p1 = host.global_plan(t.nnz, 16, host.derive_seed(host.derive_seed(1, [1]), [1]))
    p2 = host.global_plan(t.nnz, 16, host.derive_seed(host.derive_seed(1, [1]), [2]))
    upload(session, t, m)
    session.factor_phase(0, p1, 16, 1e-3, 1e-4, DET)
    session.core_phase(0, p2, 16, 1e-3, 1e-4, DET)
    ga, gb = session.download_model()
    O.COracle.factor_phase(t, m, p1, 16, 1e-3, 1e-4)
    O.COracle.core_phase(t, m, p2, 16, 1e-3, 1e-4)
    for n in range(3):
        assert bits_equal(ga[n], m.a[n]) and bits_equal(gb[n], m.b[n])


# ---------------------------------------------------------------------------
# Hogwild (throughput) mode


def planted(seed=3, nnz=60000, dims=(300, 200, 100), j=16, r=16):
    t, _, _ = synth.planted_numpy(dims, nnz, seed, j, r, 0.05)
    return O.Tensor(t.dims, t.idx, t.vals)


def init_for(t, j, r, seed=9):
    scale = host.default_init_scale(float(np.mean(np.abs(t.vals))), t.order, r, [j] * t.order)
    a, b = host.init_model(t.dims, [j] * t.order, r, seed, scale)
    return O.Model(t.dims, np.array([j] * t.order, np.int32), r, a, b)


PRECS = [eng.PREC_FP32, eng.PREC_TF32, eng.PREC_3XTF32]
# Gradient tolerance per precision: fp32 = reassociation only; 3xtf32 =
# split-tf32 C = A B (~7e-4 observed); tf32 = one pass with operands rounded
# to nearest where the engine writes them (~1.5e-3 observed on this heavily
# cancelling residual-weighted sum; truncation instead gave 4e-2).
GRAD_TOL = {eng.PREC_FP32: 2e-5, eng.PREC_3XTF32: 3e-3, eng.PREC_TF32: 1e-2}


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("jr", [16, 32])
def test_hogwild_core_gradient_matches_oracle(session, prec, jr):
    """The core sweep reads the model only, so its gradient is an
    order-independent sum: compare with the oracle's sequential fp32 sum.
    fp32 (CUDA cores): reassociation only; tf32 (tcgen05): 10-bit mantissa
    operands, fp32 accumulate."""
    t = planted(j=jr, r=jr)
    m = init_for(t, jr, jr)
    session.set_option("precision", prec)
    upload(session, t, m)
    _, g = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
    session.set_option("precision", eng.PREC_FP32)
    mc = m.copy()
    want = O.COracle.core_phase(t, mc, host.global_plan(t.nnz, 16, 1), 16, 1e-3, 1e-4)
    tol = GRAD_TOL[prec]
    np.testing.assert_allclose(g, want, rtol=tol, atol=tol * np.abs(want).max())
    _, b = session.download_model()
    for n in range(3):
        np.testing.assert_allclose(b[n], mc.b[n], rtol=1e-5, atol=1e-7)


def test_hogwild_core_is_deterministic(session):
    # Same epoch seed => same tile -> warp assignment and an ordered CTA
    # reduction, so the Hogwild core sweep is reproducible run to run.
    for prec in PRECS:
        session.set_option("precision", prec)
        t = planted()
        m = init_for(t, 16, 16)
        upload(session, t, m)
        _, g1 = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
        upload(session, t, m)
        _, g2 = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
        assert np.array_equal(g1, g2)
    session.set_option("precision", eng.PREC_FP32)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("jr", [16, 32])
@pytest.mark.parametrize("update", [1, 0])
def test_hogwild_factor_distinct_rows_match_oracle(session, prec, jr, update):
    """With every nonzero on its own rows, Hogwild has no conflicts and each
    nonzero sees the initial model: each row's update step must match the
    oracle's (fp32: FFMA vs mul+add rounding; tf32: 10-bit operands)."""
    n = 1000
    idx = np.stack([np.arange(n), (np.arange(n) * 7) % n, (np.arange(n) * 13) % n], 1)
    vals = np.linspace(1, 5, n).astype(np.float32)
    t = O.Tensor(np.array([n, n, n], np.int32), idx.astype(np.int32), vals)
    m = init_for(t, jr, jr)
    session.set_option("precision", prec)
    session.set_option("hog_update", update)
    upload(session, t, m)
    session.factor_phase(0, None, 16, 1e-2, 1e-3, HOG, seed=3)
    session.set_option("precision", eng.PREC_FP32)
    session.set_option("hog_update", 1)
    a, _ = session.download_model()
    mc = m.copy()
    O.COracle.factor_phase(t, mc, np.arange(n), 16, 1e-2, 1e-3)
    for k in range(3):
        got, want = a[k] - m.a[k], mc.a[k] - m.a[k]
        tol = 1e-4 if prec == eng.PREC_FP32 else 2e-2
        np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.abs(want).max())


def _c1p_problem():
    cfg = synth.CONFIGS["c1"]
    c, _, _ = synth.planted_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], 16, 16, 0.1)
    (tri, trv), (tei, tev) = host.split_train_test(c.dims, c.idx, c.vals, 0.014, 7)
    scale = host.default_init_scale(float(np.mean(np.abs(trv))), 3, 16, [16] * 3)
    a, b = host.init_model(c.dims, [16] * 3, 16, host.derive_seed(1, [77]), scale)
    return c.dims, (tri, trv), (tei, tev), a, b


@pytest.mark.slow
def test_c1p_rmse_trajectory_vs_reference():
    """North-star parity on config 1 (planted values):
    50 epochs of ftk::train through the C++ API.  Deterministic mode must
    match the reference's workers=1 trajectory (tolerance 1e-3 per epoch;
    observed bit-identical), Hogwild mode must stay within 1e-3 of it."""
    z = load("c1_trajectory")
    dims, (tri, trv), (tei, tev), a0, b0 = _c1p_problem()
    assert trv.size == int(z["c1p_ntrain"])
    host.set_device_options(mode=0, precision=0, exact_eval=True)
    a, b = [x.copy() for x in a0], [x.copy() for x in b0]
    h = host.train(dims, [16] * 3, 16, tri, trv, tei, tev, a, b, epochs=50, seed=1, workers=1)
    ref = z["c1p_w1_rmse"]
    assert np.max(np.abs(h["rmse"] - ref)) < 1e-3
    assert np.array_equal(h["rmse"], ref)  # deterministic mode is bit-exact
    assert np.array_equal(h["loss"], z["c1p_w1_loss"])
    for prec in (0, 1):
        host.set_device_options(mode=2, precision=prec, exact_eval=True)
        a, b = [x.copy() for x in a0], [x.copy() for x in b0]
        hh = host.train(dims, [16] * 3, 16, tri, trv, tei, tev, a, b, epochs=50, seed=1,
                        workers=8)
        dev = np.abs(hh["rmse"] - ref)
        assert np.max(dev) < 1e-3, (prec, dev)
    host.set_device_options(mode=0, precision=0, exact_eval=True)
