"""Per-block device times of the FasterTucker / FastTucker epochs on one shape
(diagnostics for scripts/variant_speed.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402  (C cache build for the probe's input only)
import paper_2404_10087_b200 as eng  # noqa: E402
import datagen as synth  # noqa: E402
from paper_2404_10087_b200 import host  # noqa: E402
from test_fastertucker import group_by_row, plan  # noqa: E402

dims, nnz, j = [10000, 10000, 1000], 1_000_000, 16
coo = synth.uniform_numpy(dims, nnz, 1)
t = O.Tensor(np.array(dims, np.int32), coo.idx, coo.vals)
m = O.random_model(dims, [j] * 3, j, 2, 0.1)
s = eng.Session(0)
s.upload_tensor(0, t.dims, t.idx, t.vals)
s.upload_model(m.dims, m.ranks, m.r, m.a, m.b)
s.ccache_upload(O.COracle.ccache_build(m))
for factor, tag in ((True, 1), (False, 2)):
    for mode in range(3):
        perm, bo = plan(t, mode, 16, 9, tag, False)
        if factor:
            g, off = group_by_row(t, perm, mode)
            ms = s.fastertucker_factor(0, mode, g, off)
            print(f"fastertucker factor mode {mode}: {ms:.2f} ms ({off.size - 1} row chains)")
        else:
            ms = s.fastertucker_core(0, mode, perm, bo)
            ms2 = s.fastertucker_core(0, mode, perm, bo, schedule=eng.MODE_HOGWILD)
            print(f"fastertucker core mode {mode}: {ms:.2f} ms chain, {ms2:.2f} ms parallel "
                  f"({bo.size - 1} batches)")
for mode in range(3):
    perm, boff = host.per_bucket_plan(t.idx, mode, 16, 5)
    ms = s.fasttucker_factor(0, mode, perm, boff)
    print(f"fasttucker factor mode {mode}: {ms:.2f} ms ({boff.size - 1} buckets)")
for mode in range(3):
    perm = host.global_plan(nnz, 16, 6 + mode)
    for sched in (eng.MODE_DETERMINISTIC, eng.MODE_HOGWILD):
        ms = s.fasttucker_core(0, mode, perm, 16, schedule=sched)
        print(f"fasttucker core mode {mode} sched {sched}: {ms:.2f} ms")
