import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
import paper_2404_10087_b200 as eng
import datagen as synth
from paper_2404_10087_b200 import host
s = eng.Session(0)
for jr in (16, 32):
    t, _, _ = synth.planted_numpy((300, 200, 100), 60000, 3, jr, jr, 0.05)
    scale = host.default_init_scale(float(np.mean(np.abs(t.vals))), 3, jr, [jr] * 3)
    a, b = host.init_model(t.dims, [jr] * 3, jr, 9, scale)
    m = O.Model(t.dims, np.array([jr] * 3, np.int32), jr, a, b)
    want = O.COracle.core_phase(O.Tensor(t.dims, t.idx, t.vals), m.copy(), host.global_plan(t.nnz, 16, 1), 16, 1e-3, 1e-4)
    for prec in (0, 1, 2):
        s.set_option("precision", prec)
        s.upload_tensor(0, t.dims, t.idx, t.vals)
        s.upload_model(t.dims, [jr] * 3, jr, a, b)
        _, g = s.core_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=5, want_grad=True)
        err = np.abs(g - want).max() / np.abs(want).max()
        print(f"J=R={jr} prec {prec} grad rel err {err:.3e}", flush=True)
