"""Test-RMSE trajectories at the headline configuration under engine options,
against the reference trajectory (tests/golden/c2_trajectory.json).

    python scripts/c2_rmse_probe.py uniform "precision=1" "precision=1,max_ctas=16" ...

Each argument after the value model is one run: comma-separated
ftkcu_set_option key=value pairs.  Prints one JSON line per run.
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
import paper_2404_10087_b200 as eng  # noqa: E402
from paper_2404_10087_b200 import host  # noqa: E402


def main():
    kind = sys.argv[1]
    runs = sys.argv[2:] or ["precision=1"]
    with open(os.path.join(ROOT, "tests", "golden", "c2_trajectory.json")) as f:
        ref = json.load(f)[kind]
    _, j, tr, te = datagen.workload("netflix", 0, kind, 0)
    order = tr.order
    scale = host.default_init_scale(float(np.mean(np.abs(tr.vals.astype(np.float64)))), order, j,
                                    [j] * order)
    a0, b0 = host.init_model(tr.dims, [j] * order, j, host.derive_seed(1, [77]), scale)
    s = eng.Session(0)
    s.set_option("eval", eng.EVAL_FAST)
    s.upload_tensor(0, tr.dims, tr.idx, tr.vals)
    s.upload_tensor(1, te.dims, te.idx, te.vals)
    want = [ref["rmse_init"]] + ref["rmse"]
    for run in runs:
        opts = dict(kv.split("=") for kv in run.split(",") if kv)
        for k, v in opts.items():
            s.set_option(k, int(v))
        s.upload_model(tr.dims, [j] * order, j, [x.copy() for x in a0], [x.copy() for x in b0])
        ev = s.eval(1, 1, 0.0, 0.0)
        rm = [float(np.sqrt(ev[0] / te.nnz))]
        t0 = time.time()
        ms = []
        for e in range(len(ref["rmse"])):
            es = host.derive_seed(1, [e + 1])
            f = s.factor_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD,
                               seed=host.derive_seed(es, [1]))
            c = s.core_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD,
                             seed=host.derive_seed(es, [2]))
            ms.append([f, c])
            ev = s.eval(1, 1, 0.0, 0.0)
            rm.append(float(np.sqrt(ev[0] / te.nnz)))
        dev = [x - y for x, y in zip(rm, want)]
        print(json.dumps({"kind": kind, "opts": opts, "engine": rm, "reference": want,
                          "delta": dev, "max_abs": max(abs(x) for x in dev), "ms": ms,
                          "kernels": [s.get_option("last_factor_kernel"),
                                      s.get_option("last_core_kernel")],
                          "wall": time.time() - t0}), flush=True)
        for k in opts:  # back to defaults
            s.set_option(k, {"precision": 1, "max_ctas": 0, "staleness": 32, "hog_update": 1,
                             "core16": 2, "tc_ws": 1}.get(k, 0))
    s.close()


if __name__ == "__main__":
    main()
