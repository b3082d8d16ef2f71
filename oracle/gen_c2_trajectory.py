"""Reference RMSE trajectories at the headline configuration (BASELINE.json
configs[1]: Netflix-shaped 480189 x 17770 x 2182, 99,072,112 training
nonzeros, J = R = 32, M = 16, reference default hyperparameters).

TEST INFRASTRUCTURE ONLY (needs oracle/_ref and a GPU for the tensor
generator, so it runs on the GPU box).  For each value model -- "uniform"
(U[1,5], the benchmark data) and "planted" (a J = R = 32 FastTucker model
plus N(0, 0.1^2) on the same tuples, so the RMSE moves) -- it regenerates the
exact tensors bench.py times (datagen.workload), initialises the model as the
reference CLI does (ftk.cpp:169-173: default_init_scale over the training
values, init_model with derive_seed(1, {77})) and runs ftkref::train
(decomposition.cpp:849-917) with workers = this host's cores for EPOCHS
epochs, test RMSE/MAE per epoch (evaluation.cpp:56-72).  The result, with a
content fingerprint of each generated tensor, goes to
tests/golden/c2_trajectory.json; bench.py compares the engine's trajectory
with it (test_rmse_vs_reference).

    python oracle/gen_c2_trajectory.py [epochs]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c2_trajectory.json")


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["planted", "uniform"]
    R = O.REF
    workers = os.cpu_count() or 1
    out = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out = json.load(f)
    for kind in kinds:
        t0 = time.time()
        cfg, j, tr, te = datagen.workload("netflix", 0, kind, 0)
        fp = datagen.fingerprint(tr)
        t_gen = time.time() - t0
        order = tr.order
        ranks = [j] * order
        scale = R.default_init_scale(float(np.mean(np.abs(tr.vals.astype(np.float64)))), order,
                                     j, ranks)
        m0 = R.init_model(tr.dims, ranks, j, R.derive_seed(1, [77]), scale)
        trt = O.Tensor(tr.dims, tr.idx, tr.vals)
        tet = O.Tensor(te.dims, te.idx, te.vals)
        rmse0, mae0 = R.evaluate(m0, tet, workers)
        t1 = time.time()
        h = R.train(trt, tet, m0, epochs=epochs, seed=1, workers=workers)
        out[kind] = {
            "workload": "netflix", "values": kind, "dims": [int(d) for d in tr.dims],
            "nnz_train": int(tr.nnz), "nnz_test": int(te.nnz), "J": j, "R": j, "M": 16,
            "lr_a": 1e-3, "lr_b": 1e-3, "reg_a": 1e-4, "reg_b": 1e-4, "seed": 1,
            "init_seed": int(R.derive_seed(1, [77])), "init_scale": float(scale),
            "workers": workers, "fingerprint_train": fp,
            "rmse_init": float(rmse0), "mae_init": float(mae0),
            "rmse": [float(x) for x in h["rmse"]], "mae": [float(x) for x in h["mae"]],
            "loss": [float(x) for x in h["loss"]],
            "epoch_seconds": [float(x) for x in h["seconds"]],
            "generator_seconds": t_gen, "train_seconds": time.time() - t1,
        }
        print(kind, json.dumps(out[kind]), flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
