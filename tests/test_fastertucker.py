"""FasterTucker baseline: complement-keyed samplers and
the oracle's factor / core blocks (with the C cache) against the reference.

Golden fixtures (tests/golden/fastertucker_*.npz, generated from the
unmodified reference by oracle/gen_golden.py) always run; the live checks
need oracle/_ref.
"""
import numpy as np
import pytest

import oracle as O
from golden_io import bits_equal, load, model, names, tensor
from paper_2404_10087_b200 import host

CO = O.COracle
needs_ref = pytest.mark.skipif(O.REF is None, reason="reference library not built")


def batch_offsets(boff, cap):
    """Batches cut from each bucket in cap-entry chunks (EpochPlan::per_bucket)."""
    out = []
    for b in range(boff.size - 1):
        out.extend(range(int(boff[b]), int(boff[b + 1]), cap))
    out.append(int(boff[-1]))
    return np.array(out, np.int64)


def plan(t, mode, cap, seed, tag, canonical):
    """(positions, batch offsets) of the block's plan: the complement-keyed
    per-bucket plan, or storage order with one entry per batch."""
    if canonical:
        return np.arange(t.nnz, dtype=np.int64), np.arange(t.nnz + 1, dtype=np.int64)
    perm, boff = host.per_bucket_plan(t.idx, mode, cap, host.derive_seed(seed, [tag, mode]), 1)
    return perm, batch_offsets(boff, cap)


def group_by_row(t, perm, mode):
    """The device factor block's input: plan positions regrouped by mode-n row
    (plan order kept inside a row) and the group offsets."""
    order = np.argsort(t.idx[perm, mode], kind="stable")
    g = perm[order]
    keys = t.idx[g, mode]
    cuts = np.flatnonzero(np.diff(keys)) + 1
    return g, np.concatenate([[0], cuts, [g.size]]).astype(np.int64)


def oracle_epoch(t, m, seed, cap, canonical, lr_a, lr_b, reg_a, reg_b):
    cache = CO.ccache_build(m)
    for factor, lr, reg, tag in ((True, lr_a, reg_a, 1), (False, lr_b, reg_b, 2)):
        for mode in range(t.order):
            perm, bo = plan(t, mode, cap, seed, tag, canonical)
            CO.fastertucker_block(factor, t, m, cache, perm, bo, mode, lr, reg)
    return cache


@pytest.mark.parametrize("name", names("fastertucker_"))
def test_complement_plans_match_golden(name):
    z = load(name)
    t, cap, seed = tensor(z), int(z["cap"]), int(z["seed"])
    for n in range(t.order):
        for tag in (1, 2):
            perm, boff = host.per_bucket_plan(t.idx, n, cap, host.derive_seed(seed, [tag, n]), 1)
            assert np.array_equal(perm, z[f"plan{tag}_{n}"])
            assert np.array_equal(boff, z[f"boff{tag}_{n}"])
            # a bucket shares every index but mode n's, which are distinct in it
            other = np.delete(t.idx[perm], n, axis=1)
            for b in range(boff.size - 1):
                seg = slice(boff[b], boff[b + 1])
                assert np.all(other[seg] == other[boff[b]])
                assert np.unique(t.idx[perm[seg], n]).size == boff[b + 1] - boff[b]


@pytest.mark.parametrize("name", names("fastertucker_"))
def test_oracle_epoch_matches_golden(name):
    z = load(name)
    t, m = tensor(z), model(z, "m_")
    lr_a, lr_b, reg_a, reg_b = (float(x) for x in z["hp"])
    oracle_epoch(t, m, int(z["seed"]), int(z["cap"]), bool(z["canonical"]), lr_a, lr_b, reg_a,
                 reg_b)
    want = model(z, "new_")
    for n in range(m.order):
        assert bits_equal(m.a[n], want.a[n]), f"A{n}"
        assert bits_equal(m.b[n], want.b[n]), f"B{n}"


def test_row_grouping_keeps_plan_order():
    t = O.random_tensor([20, 15, 10], 600, 8, 1.0, 5.0)
    perm, _ = plan(t, 0, 4, 3, 1, False)
    g, off = group_by_row(t, perm, 0)
    rank = np.empty(t.nnz, np.int64)
    rank[perm] = np.arange(t.nnz)
    for k in range(off.size - 1):
        seg = g[off[k]:off[k + 1]]
        assert np.all(t.idx[seg, 0] == t.idx[seg[0], 0])
        assert np.all(np.diff(rank[seg]) > 0)


@needs_ref
def test_oracle_epoch_matches_reference_live():
    t = O.random_tensor([25, 15, 12], 900, 3, 1.0, 5.0)
    m = O.random_model(t.dims, [12, 8, 16], 10, 4, 0.4)
    new, _ = O.REF.epoch_fastertucker(t, m, 4242, 1e-2, 1e-2, 1e-3, 1e-3, 3, 1)
    got = m.copy()
    oracle_epoch(t, got, 4242, 3, False, 1e-2, 1e-2, 1e-3, 1e-3)
    for n in range(t.order):
        assert bits_equal(got.a[n], new.a[n]) and bits_equal(got.b[n], new.b[n])
