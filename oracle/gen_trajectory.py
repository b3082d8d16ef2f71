"""Generates the config-1 RMSE-trajectory fixtures from the reference itself.

TEST INFRASTRUCTURE ONLY (needs oracle/_ref).  Config 1 of BASELINE.json:
10k x 10k x 1k, 1M nnz, J = R = 16, split 0.014 (986,000 train / 14,000 test),
model init as the reference CLI does it (ftk.cpp:169-173).  Two value
models: "c1" (uniform U[1,5], the BASELINE config) and "c1p" (planted
FastTucker J = R = 16 + N(0, 0.1^2), so the trajectory
moves).  The tensors are regenerated bit-identically from their numpy seeds
on the GPU box; only the trajectories are committed.

    python oracle/gen_trajectory.py [epochs]
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


def problem(kind):
    cfg = synth.CONFIGS["c1"]
    if kind == "c1":
        t = synth.uniform_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], cfg["lo"], cfg["hi"])
    else:
        t, _, _ = synth.planted_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], 16, 16, 0.1)
    return O.Tensor(t.dims, t.idx, t.vals)


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    R = O.REF
    out = {}
    for kind in ("c1p", "c1"):
        full = problem(kind)
        tr, te = R.split(full, 0.014, 7)
        ranks, r = [16, 16, 16], 16
        scale = R.default_init_scale(float(np.mean(np.abs(tr.vals))), 3, r, ranks)
        m0 = R.init_model(full.dims, ranks, r, derive_seed(1, [77]), scale)
        for workers in (1, 8):
            ep = epochs if (kind == "c1p" or workers == 8) else min(epochs, 10)
            t0 = time.time()
            h = R.train(tr, te, m0, epochs=ep, seed=1, workers=workers)
            print(kind, workers, ep, f"{time.time() - t0:.1f}s", h["rmse"][:3], h["rmse"][-1],
                  flush=True)
            for k in ("loss", "rmse", "mae", "seconds"):
                out[f"{kind}_w{workers}_{k}"] = h[k]
            out[f"{kind}_w{workers}_reads"] = h["reads"]
            out[f"{kind}_w{workers}_mults"] = h["mults"]
        out[f"{kind}_scale"] = np.float32(scale)
        out[f"{kind}_ntrain"] = np.int64(tr.nnz)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c1_trajectory.npz"), **out)


if __name__ == "__main__":
    main()
