"""Dev experiment: Hogwild test-RMSE trajectory on config 1 (planted) vs the
reference's workers=1 / workers=8 trajectories (tests/golden/c1_trajectory.npz)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_10087_b200 as eng
import datagen as synth
from paper_2404_10087_b200 import host

z = dict(np.load("tests/golden/c1_trajectory.npz"))
cfg = synth.CONFIGS["c1"]
kind = sys.argv[1] if len(sys.argv) > 1 else "c1p"
if kind == "c1p":
    c, _, _ = synth.planted_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], 16, 16, 0.1)
else:
    c = synth.uniform_numpy(cfg["dims"], cfg["nnz"], cfg["seed"], cfg["lo"], cfg["hi"])
(tri, trv), (tei, tev) = host.split_train_test(c.dims, c.idx, c.vals, 0.014, 7)
scale = host.default_init_scale(float(np.mean(np.abs(trv))), 3, 16, [16] * 3)
a0, b0 = host.init_model(c.dims, [16] * 3, 16, host.derive_seed(1, [77]), scale)
s = eng.Session(0)
s.set_option("eval", eng.EVAL_FAST)
ep = len(z[f"{kind}_w8_rmse"])
for upd in (1, 0):
    for prec in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"])]:
        s.set_option("hog_update", upd)
        s.set_option("precision", prec)
        s.upload_tensor(0, c.dims, tri, trv); s.upload_tensor(1, c.dims, tei, tev)
        s.upload_model(c.dims, [16] * 3, 16, a0, b0)
        rm = []; t0 = time.time()
        for e in range(1, ep + 1):
            es = host.derive_seed(1, [e])
            s.factor_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=host.derive_seed(es, [1]))
            s.core_phase(0, None, 16, 1e-3, 1e-4, eng.MODE_HOGWILD, seed=host.derive_seed(es, [2]))
            o = s.eval(1, 1); rm.append(np.sqrt(o[0] / tev.size))
        rm = np.array(rm)
        d1 = np.abs(rm - z[f"{kind}_w1_rmse"][:ep]) if f"{kind}_w1_rmse" in z and len(z[f"{kind}_w1_rmse"]) >= ep else np.abs(rm[:len(z[f"{kind}_w1_rmse"])] - z[f"{kind}_w1_rmse"])
        d8 = np.abs(rm - z[f"{kind}_w8_rmse"][:ep])
        print(f"{kind} update={upd} prec={prec} {time.time()-t0:.1f}s max|d_w1|={d1.max():.2e} max|d_w8|={d8.max():.2e} first={rm[:3]} last={rm[-1]:.6f}", flush=True)
