"""How far the reference's own test-RMSE trajectory moves with its worker
count at the headline configuration (Netflix shape, J = R = 32, uniform
values, reference default hyperparameters).

TEST INFRASTRUCTURE ONLY.  ftkref::train (decomposition.cpp:849-917) is
Hogwild for workers > 1 with the overwrite row rule (decomposition.cpp:268),
so its trajectory on unlearnable (uniform) values depends on how many
batches are in flight.  This runs it on one tensor for several worker
counts and writes the trajectories to tests/golden/c2_workers_spread.json,
which bench.py reports beside the engine-vs-reference delta.

The tensor is datagen.workload("netflix", device="cpu"): the same generator
and split as the bench tensor but torch's CPU random stream, so it is a
statistically equivalent tensor, not the bench's bytes (its fingerprint is
recorded).  Runs on CPU (no GPU needed):

    python oracle/ref_workers_spread.py EPOCHS W1,W2,...
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

OUT = os.path.join(ROOT, "tests", "golden", "c2_workers_spread.json")


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    workers = [int(w) for w in (sys.argv[2] if len(sys.argv) > 2 else "1").split(",")]
    R = O.REF
    t0 = time.time()
    cfg, j, tr, te = datagen.workload("netflix", 0, "uniform", "cpu")
    fp = datagen.fingerprint(tr)
    t_gen = time.time() - t0
    order = tr.order
    ranks = [j] * order
    scale = R.default_init_scale(float(np.mean(np.abs(tr.vals.astype(np.float64)))), order, j,
                                 ranks)
    trt = O.Tensor(tr.dims, tr.idx, tr.vals)
    tet = O.Tensor(te.dims, te.idx, te.vals)
    for w in workers:
        m0 = R.init_model(tr.dims, ranks, j, R.derive_seed(1, [77]), scale)
        rmse0, _ = R.evaluate(m0, tet, 8)
        t1 = time.time()
        h = R.train(trt, tet, m0, epochs=epochs, seed=1, workers=w)
        rec = {"workload": "netflix", "values": "uniform", "tensor": "datagen cpu stream",
               "fingerprint_train": fp, "nnz_train": int(tr.nnz), "nnz_test": int(te.nnz),
               "J": j, "R": j, "M": 16, "lr_a": 1e-3, "lr_b": 1e-3, "reg_a": 1e-4,
               "reg_b": 1e-4, "seed": 1, "workers": w, "rmse_init": float(rmse0),
               "rmse": [float(x) for x in h["rmse"]],
               "epoch_seconds": [float(x) for x in h["seconds"]],
               "generator_seconds": t_gen, "train_seconds": time.time() - t1}
        print(json.dumps(rec), flush=True)
        out = {}
        if os.path.exists(OUT):
            with open(OUT) as f:
                out = json.load(f)
        out[str(w)] = rec
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
