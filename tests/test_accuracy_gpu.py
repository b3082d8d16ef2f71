"""Accuracy of the Hogwild tensor-core sweeps the benchmark runs, against the
reference's update rule (VERDICT r01 "next" item 1).

* Row collisions.  One 128-nonzero tile over ALL cells of a tiny tensor, so
  every factor row receives 16-32 updates in the same tile.  A tile's rows
  are gathered once (the snapshot) and its steps are summed into the rows
  (RED.ADD): that is the accumulate rule, restated here in fp64 --
  A_n[i] += sum_{m: idx_n[m] = i} lr (r_m u_m - reg a_i), with u_m, r_m from
  the snapshot (decomposition.cpp:254-275 for one nonzero's step).
* Regulariser.  The same check with reg_a large enough that lr reg a
  dominates lr r u, so a missing or sign-flipped regulariser GEMM fails
  (at reg = 1e-3 it is ~6e-4 of the step and hides in the tolerance).
* Both for every factor kernel the engine dispatches (asserted through
  get_option("last_factor_kernel")), and for the overwrite rule on distinct
  rows.
* The J = R = 32 planted RMSE trajectory: ftk::train through the headline
  kernels (ws_factor_kernel + ws_core16_kernel) within 1e-3 of the
  reference's workers = 1 trajectory at every epoch
  (tests/golden/c1p32_trajectory.npz, oracle/gen_trajectory32.py).

Tolerances are per element, from a first-order error model of the
arithmetic: each contribution's step carries relative operand error eps
(tf32: 10-bit mantissa; the residual inherits eps |x_hat| from the C GEMM),
so |got - want| <= sum_m lr (eps (|r_m| + |x_hat_m|) |u_m| + eps reg |a|).
No max-based atol.
"""
import numpy as np
import pytest

import oracle as O
import paper_2404_10087_b200 as eng
from golden_io import load
import datagen as synth
from paper_2404_10087_b200 import host

pytestmark = pytest.mark.gpu
HOG = eng.MODE_HOGWILD

# relative operand error per precision (fp32: FFMA vs mul+add reassociation)
EPS = {eng.PREC_FP32: 2e-6, eng.PREC_TF32: 4e-3, eng.PREC_3XTF32: 4e-5}


def _cells_tensor(dims, nnz, seed):
    """nnz distinct cells of a tensor with prod(dims) >= nnz cells."""
    rng = np.random.default_rng(seed)
    cells = int(np.prod(dims))
    keys = rng.permutation(cells)[:nnz]
    idx = np.stack(np.unravel_index(keys, dims), 1).astype(np.int32)
    vals = rng.uniform(1.0, 5.0, nnz).astype(np.float32)
    return O.Tensor(np.array(dims, np.int32), idx, vals)


def _model(t, j, r, seed=9):
    scale = host.default_init_scale(float(np.mean(np.abs(t.vals))), t.order, r, [j] * t.order)
    a, b = host.init_model(t.dims, [j] * t.order, r, seed, scale)
    return O.Model(t.dims, np.array([j] * t.order, np.int32), r, a, b)


def _predict(m, idx):
    prod = None
    for n in range(len(m.a)):
        c = m.a[n].astype(np.float64)[idx[:, n]] @ m.b[n].astype(np.float64)
        prod = c if prod is None else prod * c
    return prod.sum(1)


def accumulate_rule(t, m, lr, reg, eps):
    """fp64 accumulate-rule step of one tile from the snapshot m, plus the
    per-element error bound and the |r u| / |reg a| contribution sums."""
    order = t.order
    a = [x.astype(np.float64) for x in m.a]
    b = [x.astype(np.float64) for x in m.b]
    rows = [a[n][t.idx[:, n]] for n in range(order)]
    c = [rows[n] @ b[n] for n in range(order)]  # [nnz, R]
    prod = np.prod(np.stack(c), axis=0)
    xhat = prod.sum(1)
    r = t.vals.astype(np.float64) - xhat
    delta = [np.zeros_like(x) for x in a]
    bound = [np.zeros_like(x) for x in a]
    ru_sum = [np.zeros_like(x) for x in a]
    ra_sum = [np.zeros_like(x) for x in a]
    for n in range(order):
        d = np.ones_like(c[0])
        for k in range(order):
            if k != n:
                d *= c[k]
        u = d @ b[n].T  # [nnz, J]
        step = lr * (r[:, None] * u - reg * rows[n])
        err = lr * (eps * (np.abs(r) + np.abs(xhat))[:, None] * np.abs(u)
                    + eps * reg * np.abs(rows[n]))
        np.add.at(delta[n], t.idx[:, n], step)
        np.add.at(bound[n], t.idx[:, n], err)
        np.add.at(ru_sum[n], t.idx[:, n], lr * np.abs(r[:, None] * u))
        np.add.at(ra_sum[n], t.idx[:, n], lr * reg * np.abs(rows[n]))
    return delta, bound, ru_sum, ra_sum


# (label, order/dims, J = R, options, expected kernel)
KERNELS = [
    ("ws", (4, 8, 4), 32, dict(precision=eng.PREC_TF32), eng.K_WS),
    # one mode-3 row: every warp's rows share it, so the sweep merges them
    # into one RED per warp (the path DSGD cells in mode-3 runs take)
    ("ws-merge", (8, 16, 1), 32, dict(precision=eng.PREC_TF32), eng.K_WS),
    # the stream in last-mode runs (option runs): aligned 16-nonzero chunks
    # share their mode-3 row, so warps merge even with 4 mode-3 rows
    ("ws-runs", (8, 4, 4), 32, dict(precision=eng.PREC_TF32, runs=1), eng.K_WS),
    ("wsf", (4, 8, 4), 32, dict(precision=eng.PREC_TF32, factor_warps=16), eng.K_WSF),
    ("ws3", (4, 8, 4), 32, dict(precision=eng.PREC_3XTF32), eng.K_WS3),
    ("tc3", (4, 8, 4), 32, dict(precision=eng.PREC_3XTF32, tc_ws=0), eng.K_TC),
    ("tc", (4, 8, 4), 32, dict(precision=eng.PREC_TF32, tc_ws=0), eng.K_TC),
    # hog_factor_kernel (fp32 CUDA cores, precision=fp32 only) is absent: a
    # warp walks its tile in groups of 4 nonzeros and re-reads the live rows
    # per group, so a tile has no single snapshot and the accumulate rule
    # above does not describe it; it is checked on distinct rows below.
    ("wsg16", (4, 8, 4), 16, dict(precision=eng.PREC_TF32), eng.K_WSG),
    ("wsg8", (4, 8, 4), 8, dict(precision=eng.PREC_TF32), eng.K_WSG),
    ("wsg-order4", (4, 4, 4, 2), 16, dict(precision=eng.PREC_TF32), eng.K_WSG),
    ("big64", (4, 8, 4), 64, dict(precision=eng.PREC_TF32), eng.K_BIG),
    ("big128", (4, 8, 4), 128, dict(precision=eng.PREC_TF32), eng.K_BIG),
]
DEFAULTS = dict(precision=eng.PREC_FP32, tc_ws=1, factor_warps=8, hog_update=1, max_ctas=0,
                runs=0)


def _run_factor(session, t, m, opts, lr, reg):
    for k, v in opts.items():
        session.set_option(k, v)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        session.factor_phase(0, None, 16, lr, reg, HOG, seed=3)
        kern = session.get_option("last_factor_kernel")
        a, _ = session.download_model()
    finally:
        for k, v in DEFAULTS.items():
            session.set_option(k, v)
    return a, kern


@pytest.mark.parametrize("nnz", [128, 100], ids=["full-tile", "ragged"])
@pytest.mark.parametrize("regime", ["normal", "reg-dominant"])
@pytest.mark.parametrize("case", KERNELS, ids=[k[0] for k in KERNELS])
def test_factor_collisions_accumulate_rule(session, case, regime, nnz):
    label, dims, jr, opts, want_kernel = case
    t = _cells_tensor(dims, nnz, 11 + jr)
    m = _model(t, jr, jr)
    lr, reg = (1e-2, 1e-3) if regime == "normal" else (1e-2, 0.5)
    if regime == "reg-dominant":  # values ~ the model's own predictions: r ~ 0
        t.vals = _predict(m, t.idx) + 0.01 * np.random.default_rng(5).standard_normal(nnz)
        t.vals = t.vals.astype(np.float32)
    a, kern = _run_factor(session, t, m, opts, lr, reg)
    if want_kernel is not None:
        assert kern == want_kernel, (label, kern)
    delta, bound, ru, ra = accumulate_rule(t, m, lr, reg, EPS[opts["precision"]])
    if regime == "reg-dominant":  # the regulariser must be what the check sees
        assert sum(x.sum() for x in ra) > 3 * sum(x.sum() for x in ru)
    hit = 0
    for n in range(t.order):
        got = a[n].astype(np.float64) - m.a[n].astype(np.float64)
        # fp32 storage of a + delta: half an ulp of the result per update
        ulp = np.spacing(np.abs(m.a[n]) + np.abs(a[n])).astype(np.float64)
        tol = 1.5 * bound[n] + 64 * ulp
        bad = np.abs(got - delta[n]) > tol
        assert not bad.any(), (label, n, np.argwhere(bad)[:5], got[bad][:5], delta[n][bad][:5])
        hit += int((np.abs(delta[n]) > 0).any(axis=1).sum())
        # rows no nonzero touches stay bit-identical
        untouched = np.setdiff1d(np.arange(t.dims[n]), t.idx[:, n])
        assert np.array_equal(a[n][untouched], m.a[n][untouched])
    assert hit > 0


@pytest.mark.parametrize("regime", ["normal", "reg-dominant"])
def test_hog_factor_collisions_group_rule(session, regime):
    """hog_factor_kernel (fp32 CUDA cores) with every row colliding: a caller
    plan fixes the stream order, the one 128-nonzero tile goes to one warp,
    which steps in groups of 4 nonzeros from the LIVE rows (accumulate rule
    inside a group, groups sequential) -- restated here in fp64."""
    t = _cells_tensor((4, 8, 4), 128, 43)
    m = _model(t, 32, 32)
    lr, reg = (1e-2, 1e-3) if regime == "normal" else (1e-2, 0.5)
    if regime == "reg-dominant":
        t.vals = (_predict(m, t.idx) + 0.01 * np.random.default_rng(5).standard_normal(128)).astype(
            np.float32)
    plan = np.random.default_rng(2).permutation(128).astype(np.int64)
    session.set_option("precision", eng.PREC_FP32)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        session.factor_phase(0, plan, 16, lr, reg, HOG, seed=3)
        assert session.get_option("last_factor_kernel") == eng.K_HOG
        a, _ = session.download_model()
    finally:
        for k, v in DEFAULTS.items():
            session.set_option(k, v)
    cur = m.copy()
    cur.a = [x.astype(np.float64) for x in cur.a]
    total_bound = [np.zeros_like(x) for x in cur.a]
    for g0 in range(0, 128, 4):
        sel = plan[g0:g0 + 4]
        sub = O.Tensor(t.dims, t.idx[sel], t.vals[sel])
        delta, bound, _, _ = accumulate_rule(sub, cur, lr, reg, EPS[eng.PREC_FP32])
        for n in range(3):
            cur.a[n] = cur.a[n] + delta[n]
            total_bound[n] += bound[n]
    for n in range(3):
        got = a[n].astype(np.float64)
        ulp = np.spacing(np.abs(a[n])).astype(np.float64)
        # a sequential chain: each group's error feeds the next group's rows
        bad = np.abs(got - cur.a[n]) > 4 * total_bound[n] + 64 * ulp
        assert not bad.any(), (n, got[bad][:5], cur.a[n][bad][:5])
        assert not np.array_equal(a[n], m.a[n])


OVERWRITE = [
    ("ws", 32, dict(precision=eng.PREC_TF32, hog_update=0), eng.K_WS),
    ("tc", 32, dict(precision=eng.PREC_3XTF32, hog_update=0), eng.K_TC),
    ("tc16", 16, dict(precision=eng.PREC_TF32, hog_update=0), eng.K_TC),
    ("big64", 64, dict(precision=eng.PREC_TF32, hog_update=0), eng.K_BIG),
    ("hog", 32, dict(precision=eng.PREC_FP32, hog_update=0), eng.K_HOG),
]


@pytest.mark.parametrize("case", OVERWRITE, ids=[k[0] for k in OVERWRITE])
def test_factor_overwrite_rule_regulariser_dominant(session, case):
    """Distinct rows (no conflicts): the reference's overwrite rule
    a' = a + lr (r u - reg a) with the regulariser dominating the step."""
    label, jr, opts, want_kernel = case
    n = 1000
    idx = np.stack([np.arange(n), (np.arange(n) * 7) % n, (np.arange(n) * 13) % n], 1)
    t = O.Tensor(np.array([n, n, n], np.int32), idx.astype(np.int32),
                 np.linspace(1, 5, n).astype(np.float32))
    m = _model(t, jr, jr)
    t.vals = (_predict(m, t.idx) + 0.01 * np.random.default_rng(5).standard_normal(n)).astype(
        np.float32)
    lr, reg = 1e-2, 0.5
    a, kern = _run_factor(session, t, m, opts, lr, reg)
    if want_kernel is not None:
        assert kern == want_kernel, (label, kern)
    delta, bound, ru, ra = accumulate_rule(t, m, lr, reg, EPS[opts["precision"]])
    assert sum(x.sum() for x in ra) > 3 * sum(x.sum() for x in ru)
    for k in range(3):
        got = a[k].astype(np.float64) - m.a[k].astype(np.float64)
        ulp = np.spacing(np.abs(m.a[k]) + np.abs(a[k])).astype(np.float64)
        bad = np.abs(got - delta[k]) > 1.5 * bound[k] + 4 * ulp
        assert not bad.any(), (label, k, got[bad][:5], delta[k][bad][:5])


# ---------------------------------------------------------------------------
# J = R = 32 planted trajectory vs the reference (the benchmark's kernels)


def c1p32_problem():
    cfg = synth.CONFIGS["c1"]
    c, _, _ = synth.planted_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], 32, 32, 0.1)
    (tri, trv), (tei, tev) = host.split_train_test(c.dims, c.idx, c.vals, 0.014, 7)
    scale = host.default_init_scale(float(np.mean(np.abs(trv))), 3, 32, [32] * 3)
    a, b = host.init_model(c.dims, [32] * 3, 32, host.derive_seed(1, [77]), scale)
    return c.dims, (tri, trv), (tei, tev), a, b, scale


@pytest.mark.slow
@pytest.mark.parametrize("prec,parity", [(eng.PREC_TF32, False), (eng.PREC_3XTF32, False),
                                         (eng.PREC_TF32, True)],
                         ids=["tf32", "3xtf32", "tf32-parity"])
def test_c1p32_rmse_trajectory_vs_reference(prec, parity):
    """ftk::train, Hogwild, through the J = R = 32 kernels the headline runs:
    test RMSE within 1e-3 of the reference's workers = 1 run at EVERY epoch
    (also with ftk::DeviceOptions::parity: window 3 on half the SMs)."""
    z = load("c1p32_trajectory")
    dims, (tri, trv), (tei, tev), a0, b0, scale = c1p32_problem()
    assert trv.size == int(z["ntrain"]) and tev.size == int(z["ntest"])
    assert np.float32(scale) == z["scale"]
    ref = z["w1_rmse"]
    epochs = ref.size
    host.set_device_options(mode=2, precision=prec, exact_eval=True, parity=parity)
    try:
        a, b = [x.copy() for x in a0], [x.copy() for x in b0]
        h = host.train(dims, [32] * 3, 32, tri, trv, tei, tev, a, b, epochs=epochs, seed=1,
                       workers=8)
        kf, kc = host.last_kernels()
    finally:
        host.set_device_options(mode=0, precision=0, exact_eval=True)
    if prec == eng.PREC_TF32:
        assert (kf, kc) == (eng.K_WS, eng.K_WS16)
    else:
        assert (kf, kc) == (eng.K_WS3, eng.K_WS)
    dev = np.abs(h["rmse"] - ref)
    assert np.max(dev) < 1e-3, dev
    # the trajectory must actually move, or the check says nothing
    assert ref[0] - ref[-1] > 1e-2


@pytest.mark.slow
def test_c1p32_deterministic_prefix_bit_exact():
    """Deterministic mode at J = R = 32: the first epochs of the same run are
    bit-identical to the reference's workers = 1 trajectory."""
    z = load("c1p32_trajectory")
    dims, (tri, trv), (tei, tev), a0, b0, _ = c1p32_problem()
    host.set_device_options(mode=1, precision=0, exact_eval=True)
    try:
        a, b = [x.copy() for x in a0], [x.copy() for x in b0]
        h = host.train(dims, [32] * 3, 32, tri, trv, tei, tev, a, b, epochs=2, seed=1,
                       workers=1)
        assert host.last_kernels() == (eng.K_DET, eng.K_DET)
    finally:
        host.set_device_options(mode=0, precision=0, exact_eval=True)
    assert np.array_equal(h["rmse"], z["w1_rmse"][:2])
    assert np.array_equal(h["loss"], z["w1_loss"][:2])


# ---------------------------------------------------------------------------
# Core gradient of the J = R = 32 core sweeps, per element


def core_grad_fp64(t, m):
    """G_n[j][r] = sum_t r_t A_n[t][j] D_n[t][r] (accumulate_core_grads_plus,
    decomposition.cpp:277-296) in fp64, plus the first-order error scale
    sum_t (|r_t| + |x_hat_t|) |A_n[t][j]| |D_n[t][r]| (every operand carries
    relative error eps; the residual inherits eps |x_hat| from the C GEMM)."""
    a = [x.astype(np.float64) for x in m.a]
    b = [x.astype(np.float64) for x in m.b]
    rows = [a[n][t.idx[:, n]] for n in range(t.order)]
    c = [rows[n] @ b[n] for n in range(t.order)]
    xhat = np.prod(np.stack(c), axis=0).sum(1)
    r = t.vals.astype(np.float64) - xhat
    g, scale = [], []
    for n in range(t.order):
        d = np.ones_like(c[0])
        for k in range(t.order):
            if k != n:
                d *= c[k]
        g.append(rows[n].T @ (r[:, None] * d))
        scale.append(np.abs(rows[n]).T @ ((np.abs(r) + np.abs(xhat))[:, None] * np.abs(d)))
    return np.concatenate([x.ravel() for x in g]), np.concatenate([x.ravel() for x in scale])


@pytest.mark.parametrize("core16,max_ctas", [(1, 0), (1, 1), (1, 3), (2, 0), (2, 1), (2, 3), (0, 0)],
                         ids=["ws16", "ws16-1cta", "ws16-3cta", "ws16x2", "ws16x2-1cta", "ws16x2-3cta", "ws-tf32"])
def test_core32_gradient_per_element(session, core16, max_ctas):
    """The headline core sweep (ws_core16_kernel: fp16 copy of A, fp32
    accumulate) with one (core16 = 1) or two (core16 = 2) epilogue warp
    groups and many tiles per CTA (max_ctas = 1: all 2344 tiles on one CTA,
    both C buffers, D tiles and every ring slot reused), against the fp64
    gradient element by element."""
    c = synth.planted_numpy((300, 200, 100), 300000, 4, 32, 32, 0.05)[0]
    t = O.Tensor(c.dims, c.idx, c.vals)  # 2344 tiles: 16 per CTA on 148 SMs
    m = _model(t, 32, 32)
    session.set_option("precision", eng.PREC_TF32)
    session.set_option("core16", core16)
    session.set_option("max_ctas", max_ctas)
    try:
        session.upload_tensor(0, t.dims, t.idx, t.vals)
        session.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
        _, g = session.core_phase(0, None, 16, 1e-3, 1e-4, HOG, seed=5, want_grad=True)
        kern = session.get_option("last_core_kernel")
    finally:
        for k, v in DEFAULTS.items():
            session.set_option(k, v)
        session.set_option("core16", 2)  # the default
    assert kern == (eng.K_WS16 if core16 else eng.K_WS)
    want, scale = core_grad_fp64(t, m)
    eps = 2.0 ** -10  # fp16 / tf32 operands (10-bit mantissa), rounded to nearest
    err = np.abs(g.astype(np.float64) - want)
    bad = err > 2 * eps * scale + 1e-6 * np.abs(want).max()
    assert not bad.any(), (np.argwhere(bad)[:5], g[bad][:5], want[bad][:5])
    # the bound is meaningful: the typical error is well inside it
    assert np.median(err / (eps * scale)) < 0.5
