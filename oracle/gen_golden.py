"""Regenerates tests/golden/*.npz from the reference library itself.

TEST INFRASTRUCTURE ONLY.  Needs oracle/_ref/libftkref.so, i.e. the
unmodified reference compiled by oracle/Makefile from /root/reference (this
container).  The fixtures are small (KBs) and committed, so the oracle can be
pinned on machines without the reference tree (the GPU box).

    python oracle/gen_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2404_10087_b200.host import derive_seed  # noqa: E402  (pure Python)

OUT = os.path.join(ROOT, "tests", "golden")

# (name, dims, nnz, value range, ranks, R, cap, rows)
PROBES = [
    ("probe_j16", [9, 7, 5], 60, (0.5, 3.0), [16, 16, 16], 16, 16, list(range(16))),
    ("probe_small_ranks", [9, 7, 5], 60, (0.5, 3.0), [5, 4, 3], 4, 16, list(range(12))),
    ("probe_ragged", [9, 7, 5], 60, (0.5, 3.0), [33, 20, 8], 24, 16, list(range(5))),
    ("probe_dups", [3, 3, 2], 18, (0.0, 1.0), [4, 4, 4], 3, 16, [0, 2, 4, 6, 8, 10, 12, 14, 16,
                                                               1, 3, 5, 7, 9, 11, 13]),
    ("probe_cap7", [9, 7, 5], 60, (0.5, 3.0), [8, 8, 8], 8, 7, list(range(7))),
    ("probe_order4", [6, 5, 4, 3], 40, (1.0, 2.0), [4, 6, 4, 2], 5, 16, list(range(9))),
]

# (name, dims, nnz, ranks, R, cap, epoch seed)
EPOCHS = [
    ("epoch_j16", [30, 20, 10], 1000, [16, 16, 16], 16, 16, 1234),
    ("epoch_small", [30, 20, 10], 1000, [5, 4, 3], 4, 16, 99),
    ("epoch_cap5", [30, 20, 10], 1000, [8, 12, 4], 6, 5, 7),
    ("epoch_order5", [8, 7, 6, 5, 4], 700, [4, 4, 4, 4, 4], 4, 16, 31),
]


# Storage scheme (EpochOptions.store_c, §8 f1): same epoch fixtures with the
# core phase reading C rows from the CCache.  (name, dims, nnz, ranks, R, cap, seed)
STOREC = [
    ("storec_j16", [30, 20, 10], 1000, [16, 16, 16], 16, 16, 1234),
    ("storec_ragged", [30, 20, 10], 1000, [5, 4, 3], 4, 16, 99),
    ("storec_order4", [9, 8, 7, 6], 800, [8, 4, 8, 4], 8, 9, 5),
]


def tensor_fields(t):
    return dict(dims=t.dims, idx=t.idx, vals=t.vals)


def model_fields(m, prefix):
    out = {f"{prefix}dims": m.dims, f"{prefix}ranks": m.ranks, f"{prefix}r": np.int32(m.r)}
    for n in range(m.order):
        out[f"{prefix}a{n}"] = m.a[n]
        out[f"{prefix}b{n}"] = m.b[n]
    return out


def storec(R):
    for k, (name, dims, nnz, ranks, r, cap, seed) in enumerate(STOREC):
        t = O.random_tensor(dims, nnz, 600 + k, 1.0, 5.0)
        m = O.random_model(dims, ranks, r, 700 + k, 0.3)
        hp = dict(lr_a=1e-2, lr_b=1e-2, reg_a=1e-3, reg_b=1e-3)
        new, _, cnt = R.epoch_plus(t, m, seed, batch=cap, workers=1, store_c=True, **hp)
        p1 = R.global_plan(t.nnz, cap, derive_seed(seed, [1]))
        p2 = R.global_plan(t.nnz, cap, derive_seed(seed, [2]))
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **tensor_fields(t),
                            **model_fields(m, "m_"), **model_fields(new, "new_"),
                            cap=np.int32(cap), seed=np.uint64(seed), plan1=p1, plan2=p2,
                            counters=cnt, hp=np.array(list(hp.values()), np.float32))


# FastTucker baseline (§8 f4): (name, dims, nnz, ranks, R, cap, seed, canonical)
FASTTUCKER = [
    ("fasttucker_j16", [30, 20, 10], 1000, [16, 16, 16], 16, 16, 1234, False),
    ("fasttucker_ragged", [30, 20, 10], 1000, [5, 4, 3], 4, 16, 99, False),
    ("fasttucker_cap5", [30, 20, 10], 1000, [8, 12, 4], 6, 5, 7, False),
    ("fasttucker_order4", [9, 8, 7, 6], 800, [8, 4, 8, 4], 8, 9, 5, False),
    ("fasttucker_canonical", [20, 15, 10], 500, [8, 8, 8], 8, 16, 3, True),
]


def fasttucker(R):
    for k, (name, dims, nnz, ranks, r, cap, seed, canon) in enumerate(FASTTUCKER):
        t = O.random_tensor(dims, nnz, 800 + k, 1.0, 5.0)
        m = O.random_model(dims, ranks, r, 900 + k, 0.3)
        hp = dict(lr_a=1e-2, lr_b=1e-2, reg_a=1e-3, reg_b=1e-3)
        new, cnt = R.epoch_fasttucker(t, m, seed, batch=cap, workers=1, canonical=canon, **hp)
        plans = {}
        for n in range(t.order):  # the reference's own sampler streams
            perm, boff = R.per_bucket_plan(t, n, cap, derive_seed(seed, [1, n]))
            plans[f"fplan{n}"], plans[f"fboff{n}"] = perm, boff
            plans[f"cplan{n}"] = R.global_plan(t.nnz, cap, derive_seed(seed, [2, n]))
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **tensor_fields(t),
                            **model_fields(m, "m_"), **model_fields(new, "new_"),
                            cap=np.int32(cap), seed=np.uint64(seed), canonical=np.int32(canon),
                            counters=cnt, hp=np.array(list(hp.values()), np.float32), **plans)


# FasterTucker baseline (§8 f4): (name, dims, nnz, ranks, R, cap, seed, canonical)
FASTERTUCKER = [
    ("fastertucker_j16", [30, 20, 10], 1000, [16, 16, 16], 16, 16, 1234, False),
    ("fastertucker_ragged", [8, 6, 5], 200, [5, 4, 3], 4, 2, 99, False),
    ("fastertucker_cap5", [30, 20, 10], 1000, [8, 12, 4], 6, 5, 7, False),
    ("fastertucker_order4", [6, 5, 4, 3], 300, [4, 6, 4, 2], 5, 16, 5, False),
    ("fastertucker_canonical", [20, 15, 10], 500, [8, 8, 8], 8, 16, 3, True),
]


def fastertucker(R):
    for k, (name, dims, nnz, ranks, r, cap, seed, canon) in enumerate(FASTERTUCKER):
        t = O.random_tensor(dims, nnz, 850 + k, 1.0, 5.0)
        m = O.random_model(dims, ranks, r, 950 + k, 0.3)
        hp = dict(lr_a=1e-2, lr_b=1e-2, reg_a=1e-3, reg_b=1e-3)
        new, cnt = R.epoch_fastertucker(t, m, seed, batch=cap, workers=1, canonical=canon, **hp)
        plans = {}
        for n in range(t.order):  # the reference's complement-keyed sampler streams
            for tag in (1, 2):
                perm, boff = R.per_bucket_plan(t, n, cap, derive_seed(seed, [tag, n]), keying=1)
                plans[f"plan{tag}_{n}"], plans[f"boff{tag}_{n}"] = perm, boff
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **tensor_fields(t),
                            **model_fields(m, "m_"), **model_fields(new, "new_"),
                            cap=np.int32(cap), seed=np.uint64(seed), canonical=np.int32(canon),
                            counters=cnt, hp=np.array(list(hp.values()), np.float32), **plans)


def train_variants(R):
    """Short train() trajectories of the convex baselines (variant 1, 2)."""
    full = O.random_tensor([30, 25, 20], 2500, 510, 1.0, 5.0)
    tr, te = R.split(full, 0.1, 9)
    ranks, r = [8, 8, 8], 8
    scale = R.default_init_scale(float(np.mean(np.abs(tr.vals))), 3, r, ranks)
    m0 = R.init_model(full.dims, ranks, r, derive_seed(2, [77]), scale)
    for variant, name in ((1, "fasttucker"), (2, "fastertucker")):
        hist = R.train(tr, te, m0, epochs=3, seed=2, workers=1, variant=variant)
        np.savez_compressed(os.path.join(OUT, f"train_{name}.npz"), full_dims=full.dims,
                            tr_idx=tr.idx, tr_vals=tr.vals, te_idx=te.idx, te_vals=te.vals,
                            **model_fields(m0, "m0_"), **model_fields(hist["model"], "final_"),
                            loss=hist["loss"], rmse=hist["rmse"], mae=hist["mae"],
                            reads=hist["reads"], mults=hist["mults"])


def main():
    R = O.REF
    if R is None:
        raise SystemExit("oracle/_ref/libftkref.so missing: run make -C oracle first")
    os.makedirs(OUT, exist_ok=True)
    if "--fasttucker-only" in sys.argv:
        fasttucker(R)
        fastertucker(R)
        train_variants(R)
        return
    storec(R)
    fasttucker(R)
    fastertucker(R)
    train_variants(R)
    if "--storec-only" in sys.argv:
        return
    lr_a, reg_a = 0.05, 0.01
    for k, (name, dims, nnz, (lo, hi), ranks, r, cap, rows) in enumerate(PROBES):
        t = O.random_tensor(dims, nnz, 100 + k, lo, hi)
        m = O.random_model(dims, ranks, r, 200 + k)
        m_after = m.copy()
        out = R.batch_probe(t, m_after, rows, cap, lr_a, reg_a)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **tensor_fields(t),
                            **model_fields(m, "m_"), rows=np.array(rows, np.int64),
                            cap=np.int32(cap), lr_a=np.float32(lr_a), reg_a=np.float32(reg_a),
                            **{f"out_{key}": v for key, v in out.items()},
                            **{f"after_a{n}": m_after.a[n] for n in range(m.order)})
    for k, (name, dims, nnz, ranks, r, cap, seed) in enumerate(EPOCHS):
        t = O.random_tensor(dims, nnz, 300 + k, 1.0, 5.0)
        m = O.random_model(dims, ranks, r, 400 + k, 0.3)
        hp = dict(lr_a=1e-2, lr_b=1e-2, reg_a=1e-3, reg_b=1e-3)
        new, _, cnt = R.epoch_plus(t, m, seed, batch=cap, workers=1, **hp)
        p1 = R.global_plan(t.nnz, cap, derive_seed(seed, [1]))
        p2 = R.global_plan(t.nnz, cap, derive_seed(seed, [2]))
        loss1 = R.loss(new, t, 1e-3, 2e-3, 1)
        loss3 = R.loss(new, t, 1e-3, 2e-3, 3)
        ev1 = R.evaluate(new, t, 1)
        ev4 = R.evaluate(new, t, 4)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **tensor_fields(t),
                            **model_fields(m, "m_"), **model_fields(new, "new_"),
                            cap=np.int32(cap), seed=np.uint64(seed), plan1=p1, plan2=p2,
                            counters=cnt, hp=np.array(list(hp.values()), np.float32),
                            loss_w1=np.float64(loss1), loss_w3=np.float64(loss3),
                            eval_w1=np.array(ev1), eval_w4=np.array(ev4))
    # A short training trajectory with a held-out split (reference train()).
    full = O.random_tensor([40, 30, 20], 3000, 500, 1.0, 5.0)
    tr, te = R.split(full, 0.1, 7)
    ranks, r = [8, 8, 8], 8
    scale = R.default_init_scale(float(np.mean(np.abs(tr.vals))), 3, r, ranks)
    m0 = R.init_model(full.dims, ranks, r, derive_seed(1, [77]), scale)
    hist = R.train(tr, te, m0, epochs=4, seed=1, workers=1)
    np.savez_compressed(os.path.join(OUT, "train_small.npz"), full_dims=full.dims,
                        full_idx=full.idx, full_vals=full.vals, tr_idx=tr.idx, tr_vals=tr.vals,
                        te_idx=te.idx, te_vals=te.vals, scale=np.float32(scale),
                        **model_fields(m0, "m0_"), **model_fields(hist["model"], "final_"),
                        loss=hist["loss"], rmse=hist["rmse"], mae=hist["mae"],
                        reads=hist["reads"], mults=hist["mults"])
    # Sampler streams.
    np.savez_compressed(os.path.join(OUT, "plans.npz"),
                        p100_16_3=R.global_plan(100, 16, 3), p1000_16_42=R.global_plan(1000, 16, 42),
                        p37_5_9=R.global_plan(37, 5, 9))
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
