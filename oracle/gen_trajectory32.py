"""Generates the J = R = 32 planted RMSE-trajectory fixture from the reference.

TEST INFRASTRUCTURE ONLY (needs oracle/_ref).  Config-1 dims (10k x 10k x 1k,
1M nnz) with values planted from a FastTucker model at J = R = 32 plus
N(0, 0.1^2) (synth.planted_numpy), split 0.014 (seed 7), model init as the
reference CLI does it (ftk.cpp:169-173), hyperparameters at the reference
defaults (model.hpp:12-17).  This is the rank the benchmark runs (BASELINE.json
configs[1]), so the trajectory pins the kernels the headline uses
(ws_factor_kernel / ws_core16_kernel) -- config 1 itself is J = R = 16.

The reference trains with workers = 1 (bit-reproducible, the parity
target) and workers = 8 (its own Hogwild, for scale).  The tensor is
regenerated bit-identically from its numpy seeds on the GPU box; only the
trajectories are committed (tests/golden/c1p32_trajectory.npz).

    python oracle/gen_trajectory32.py [epochs]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import datagen as synth  # noqa: E402
from paper_2404_10087_b200.host import derive_seed  # noqa: E402

JR = 32


def problem():
    cfg = synth.CONFIGS["c1"]
    t, _, _ = synth.planted_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], JR, JR, 0.1)
    return O.Tensor(t.dims, t.idx, t.vals)


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    R = O.REF
    out = {}
    full = problem()
    tr, te = R.split(full, 0.014, 7)
    ranks, r = [JR] * 3, JR
    scale = R.default_init_scale(float(np.mean(np.abs(tr.vals))), 3, r, ranks)
    m0 = R.init_model(full.dims, ranks, r, derive_seed(1, [77]), scale)
    for workers in (8, 1):
        t0 = time.time()
        h = R.train(tr, te, m0, epochs=epochs, seed=1, workers=workers)
        print(workers, epochs, f"{time.time() - t0:.1f}s", h["rmse"][:3], h["rmse"][-1],
              flush=True)
        for k in ("loss", "rmse", "mae", "seconds"):
            out[f"w{workers}_{k}"] = h[k]
    out["scale"] = np.float32(scale)
    out["ntrain"] = np.int64(tr.nnz)
    out["ntest"] = np.int64(te.nnz)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c1p32_trajectory.npz"), **out)


if __name__ == "__main__":
    main()
