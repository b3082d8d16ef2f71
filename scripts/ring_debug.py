"""Two virtual ranks, one ring factor epoch each, concurrently on one GPU;
prints every rank's arrival flags and cell counters (debugging aid)."""
import os, sys, threading, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O
import paper_2404_10087_b200 as eng
from paper_2404_10087_b200 import dsgd

P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
emul = len(sys.argv) > 2 and sys.argv[2] == "emu"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 2
nnz = int(sys.argv[4]) if len(sys.argv) > 4 else 400_000
epochs = int(sys.argv[5]) if len(sys.argv) > 5 else 1
t = O.random_tensor([10000, 10000, 1000], nnz, 6, 0.0, 2.0)
m = O.random_model(t.dims, [32] * 3, 32, 5, 0.2)
lay = dsgd.make_ring_layout(t.dims, t.idx, P, K)
ss = []
for g in range(P):
    s = eng.Session(0)
    s.set_option("precision", eng.PREC_TF32)
    s.set_option("max_ctas", 148 // P)
    s.set_option("ring_timeout_ms", 300)
    s.upload_model(t.dims, m.ranks, m.r, [x.copy() for x in m.a], [x.copy() for x in m.b])
    idx, vals, off, _ = dsgd.ring_cells(lay, t.idx, t.vals, g)
    s.upload_tensor(0, t.dims, idx, vals)
    s.set_cells(0, off)
    ss.append(s)
blobs = [s.ring_export() for s in ss]
for g, s in enumerate(ss):
    if emul:
        s.ring_emulate(0)
    else:
        s.ring_connect(0, blobs[(g - 1) % P])
seeds = dsgd.DsgdTrainer(None, lay, 0, schedule="ring").cell_seeds(3)
bar = threading.Barrier(P)
res = [None] * P
def run(g):
    bar.wait()
    t0 = time.time()
    ss[g].ring_factor_epoch(0, P, g, lay.row_off[1], lay.row_off[2], seeds, 0.01, 0.01)
    bar.wait()  # all launched before anyone waits
    to = ss[g].ring_status()
    res[g] = (to, time.time() - t0)
Q = K * P
n = (P + 1) * (Q + P)
for e in range(epochs):
    th = [threading.Thread(target=run, args=(g,)) for g in range(P)]
    for x in th: x.start()
    for x in th: x.join()
    bad = any(r[0] for r in res)
    print("epoch", e, "timeouts", [hex(r[0]) for r in res], "secs %.3f" % max(r[1] for r in res))
    if bad:
        for g, s in enumerate(ss):
            f, d = s.ring_debug(max(n, P * Q))
            print("rank", g, "flags3", f[:(P + 1) * Q].reshape(P + 1, Q).tolist())
            print("  flags2", f[(P + 1) * Q:n].reshape(P + 1, P).tolist())
            print("  done ", d[:P * Q].tolist())
        break
