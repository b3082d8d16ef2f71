"""Pins the CPU oracle (oracle/ftk_oracle.c) to the reference.

1. Against the committed golden fixtures (tests/golden, generated from the
   unmodified reference library by oracle/gen_golden.py): always runs.
2. Against the reference library live (oracle/_ref/libftkref.so) on fresh
   random cases: runs where the reference was built.

Bit-exact comparisons throughout: the oracle restates the reference's fp32
rounding sequence, so there is no tolerance to hide behind.
"""
import numpy as np
import pytest

import oracle as O
from golden_io import bits_equal, load, model, names, tensor
from paper_2404_10087_b200.host import derive_seed

C = O.COracle
needs_ref = pytest.mark.skipif(O.REF is None, reason="reference library not built here")


@pytest.mark.parametrize("name", names("probe_"))
def test_probe_matches_golden(name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    out = C.batch_probe(t, m, z["rows"], int(z["cap"]), float(z["lr_a"]), float(z["reg_a"]))
    for key, v in out.items():
        assert bits_equal(v, z[f"out_{key}"]), key
    for n in range(m.order):
        assert bits_equal(m.a[n], z[f"after_a{n}"])


@pytest.mark.parametrize("name", names("epoch_"))
def test_epoch_matches_golden(name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    cap = int(z["cap"])
    C.factor_phase(t, m, z["plan1"], cap, lr_a, reg_a)
    C.core_phase(t, m, z["plan2"], cap, lr_b, reg_b)
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(m.a[n], want.a[n]), f"A{n}"
        assert bits_equal(m.b[n], want.b[n]), f"B{n}"
    # fp64 evaluation in the reference's slab order, exact.
    assert C.loss(want, t, 1e-3, 2e-3, 1) == float(z["loss_w1"])
    assert C.loss(want, t, 1e-3, 2e-3, 3) == float(z["loss_w3"])
    assert C.evaluate(want, t, 1) == tuple(z["eval_w1"])
    assert C.evaluate(want, t, 4) == tuple(z["eval_w4"])


def test_counters_closed_form_matches_golden():
    # The reference bills (m_eff + R) sum J reads, m_eff R sum J BD^T mults
    # and m_eff sum J updates per factor batch (decomposition.cpp:644-658);
    # the full-batch values are the closed forms of counters.cpp:486-491.
    z = load("epoch_j16")
    cnt = z["counters"]
    nnz, cap = int(z["vals"].size), int(z["cap"])
    sj, r = int(np.sum(z["m_ranks"])), int(z["m_r"])
    nb = -(-nnz // cap)
    p = C.predicted_costs(3, cap, r, z["m_ranks"])
    assert p[0] == (cap + r) * sj
    assert cnt[0] == (nnz + nb * r) * sj
    assert cnt[2] == nnz * r * sj
    assert cnt[3] == nnz * sj


def test_empty_core_phase_raises():
    t = O.Tensor(np.array([3, 3, 3], np.int32), np.zeros((0, 3), np.int32),
                 np.zeros(0, np.float32))
    m = O.random_model([3, 3, 3], [2, 2, 2], 2, 1)
    with pytest.raises(RuntimeError, match="empty tensor"):
        C.core_phase(t, m, np.zeros(0, np.int64), 16, 1e-3, 1e-4)


@needs_ref
@pytest.mark.parametrize("case", range(6))
def test_probe_matches_reference_live(case):
    rng = np.random.default_rng(case)
    order = int(rng.integers(3, 6))
    dims = [int(x) for x in rng.integers(2, 8, size=order)]
    t = O.random_tensor(dims, int(min(np.prod(dims), 50)), case, 0.1, 4.0)
    ranks = [int(x) for x in rng.integers(1, 40, size=order)]
    r = int(rng.integers(1, 40))
    cap = int(rng.integers(1, 33))
    rows = rng.choice(t.nnz, size=int(rng.integers(1, cap + 1)), replace=True)
    m = O.random_model(dims, ranks, r, case + 9, 0.7)
    m1, m2 = m.copy(), m.copy()
    a = C.batch_probe(t, m1, rows, cap, 0.03, 0.002)
    b = O.REF.batch_probe(t, m2, rows, cap, 0.03, 0.002)
    for k in a:
        assert bits_equal(a[k], b[k]), k
    for n in range(order):
        assert bits_equal(m1.a[n], m2.a[n])


@needs_ref
@pytest.mark.parametrize("cap", [16, 1, 9])
def test_epoch_matches_reference_live(cap):
    t = O.random_tensor([25, 15, 12], 900, cap, 1.0, 5.0)
    m = O.random_model(t.dims, [12, 8, 16], 10, cap + 1, 0.4)
    seed = 4242 + cap
    new, _, _ = O.REF.epoch_plus(t, m, seed, 1e-2, 1e-2, 1e-3, 1e-3, cap, 1)
    mc = m.copy()
    C.factor_phase(t, mc, O.REF.global_plan(t.nnz, cap, derive_seed(seed, [1])), cap, 1e-2, 1e-3)
    C.core_phase(t, mc, O.REF.global_plan(t.nnz, cap, derive_seed(seed, [2])), cap, 1e-2, 1e-3)
    for n in range(3):
        assert bits_equal(mc.a[n], new.a[n])
        assert bits_equal(mc.b[n], new.b[n])


@needs_ref
def test_plans_fixture_matches_reference_live():
    z = load("plans")
    assert np.array_equal(O.REF.global_plan(100, 16, 3), z["p100_16_3"])
    assert np.array_equal(O.REF.global_plan(37, 5, 9), z["p37_5_9"])


@pytest.mark.parametrize("name", names("storec_"))
def test_storage_scheme_epoch_matches_golden(name):
    """store_c (§8 f1): C rows from the CCache (decomposition.cpp:74-107,
    299-314) in the core phase; bit-exact against the reference's epoch."""
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    cap = int(z["cap"])
    C.factor_phase(t, m, z["plan1"], cap, lr_a, reg_a)
    C.core_phase(t, m, z["plan2"], cap, lr_b, reg_b, store_c=True)
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(m.a[n], want.a[n]), f"A{n}"
        assert bits_equal(m.b[n], want.b[n]), f"B{n}"


@needs_ref
def test_storage_scheme_matches_reference_live():
    t = O.random_tensor([25, 15, 12], 900, 3, 1.0, 5.0)
    m = O.random_model(t.dims, [12, 8, 16], 10, 4, 0.4)
    seed = 777
    new, _, _ = O.REF.epoch_plus(t, m, seed, 1e-2, 1e-2, 1e-3, 1e-3, 16, 1, store_c=True)
    mc = m.copy()
    C.factor_phase(t, mc, O.REF.global_plan(t.nnz, 16, derive_seed(seed, [1])), 16, 1e-2, 1e-3)
    C.core_phase(t, mc, O.REF.global_plan(t.nnz, 16, derive_seed(seed, [2])), 16, 1e-2, 1e-3,
                 store_c=True)
    for n in range(3):
        assert bits_equal(mc.a[n], new.a[n])
        assert bits_equal(mc.b[n], new.b[n])
