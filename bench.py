#!/usr/bin/env python
"""FastTuckerPlus epoch throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
                    [--config netflix|c1|yahoo|order6] [--rank J] [--precision fp32|tf32|3xtf32]

A step is one FastTuckerPlus epoch -- the factor sweep (Eq. 14) plus the core
sweep and core update (Eq. 15) -- over the whole synthetic tensor, in the
engine's Hogwild mode (the reference's workers > 1 semantics).  Prints one
JSON line (rank 0).  Metric: nonzeros / second / epoch.

Timing: W untimed epochs, then K epochs between CUDA events recorded on the
engine's own stream (torch.cuda.ExternalStream over the session stream),
barrier + synchronize on both sides, max over ranks.  The COO stream (16 B x
nnz per sweep, 1.6 GB at Netflix shape) is far larger than the 126 MB L2, so
no flush is needed between steps.

Multi-GPU (torchrun, N > 1, order-3 configs): DSGD stratification
(paper_2404_10087_b200/dsgd.py) -- rank g holds the nonzeros of
mode-1 block g, sweeps one cell per stratum (N*N strata), ring-shifts the
mode-2/3 blocks over NCCL and all-reduces dB in the core phase.  The total
tensor is fixed ("scaling": "strong"); `value` = all nonzeros / the slowest
rank's epoch time.  `--dsgd` runs the cell path at N = 1 as well.

`e2e` re-times the same epochs through the C-ABI from pinned host memory:
every step uploads the COO tensor and the model (H2D), runs the epoch and
downloads the model (D2H).  `cpu_baseline` times the reference library
(oracle/_ref, unmodified sources) on this host's cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--config", default="netflix", choices=["netflix", "c1", "yahoo", "order6"])
    ap.add_argument("--rank", type=int, default=0, help="override J = R")
    ap.add_argument("--precision", default="tf32", choices=["fp32", "tf32", "3xtf32"])
    ap.add_argument("--hog-update", type=int, default=1, help="1: atomic RED rows, 0: overwrite")
    ap.add_argument("--tc-ws", type=int, default=1, help="warp-specialized tcgen05 sweeps")
    ap.add_argument("--factor-warps", type=int, default=8, choices=[8, 16],
                    help="epilogue warps of the N=3 J=R=32 factor sweep")
    ap.add_argument("--core16", type=int, default=2,
                    help="tf32 core sweep on an fp16 copy of A (kind::f16, 10-bit mantissa)")
    ap.add_argument("--store-c", type=int, default=0,
                    help="core sweep storage scheme: C rows from a C cache rebuilt every core "
                         "phase (inside the timed region), EpochOptions.store_c")
    ap.add_argument("--dsgd", action="store_true",
                    help="DSGD cell path even at 1 GPU (always used for order 3 at N > 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--schedule", default="auto", choices=["auto", "strata", "ring"],
                    help="DSGD factor schedule at N > 1 (ring: mode-3 blocks passed over CUDA-IPC "
                         "peer memory inside one persistent kernel, falling back to the strata "
                         "if a wait times out; strata: P*P cell launches + NCCL shifts; auto: "
                         "the strata at N = 2, where a cell is 12M nonzeros and the stops are "
                         "cheap, the ring above)")
    ap.add_argument("--tokens", type=int, default=1, help="ring: mode-3 blocks per rank")
    ap.add_argument("--runs", type=int, default=0, choices=[-1, 0, 1],
                    help="Hogwild stream in 16-nonzero last-mode runs (session option runs)")
    ap.add_argument("--cell-order", default="runs", choices=["runs", "plain"],
                    help="DSGD cells in 16-nonzero mode-3 runs (the sweep merges a warp's "
                         "same-row updates of the small mode) or plain random order")
    ap.add_argument("--e2e-keys", default="delta", choices=["delta", "packed", "int32"],
                    help="COO index format on the host-to-device link in the e2e loop")
    ap.add_argument("--delta-decode", type=int, default=0, choices=[0, 1],
                    help="delta-coded e2e uploads: 0 decode beside the running epochs, 1 at "
                         "first use on the session stream (session option delta_decode)")
    ap.add_argument("--e2e-sync", action="store_true",
                    help="e2e without the double-buffered asynchronous tensor upload")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp32-equiv", action="store_true",
                    help="skip the 3xtf32 (fp32-equivalent) timing of the same epochs")
    ap.add_argument("--no-rmse-check", action="store_true",
                    help="skip the test-RMSE trajectory against tests/golden/c2_trajectory.json")
    ap.add_argument("--cpu-sample", type=int, default=4_000_000)
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: NVML polled every 2 ms from a thread (nvidia-smi's 100 ms loop
    would see one sample of a 70 ms region); nvidia-smi when NVML is absent."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.thread = None
        self.nvml = None  # (module, handle, max SM MHz, reason bits)
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)

    def poll(self):
        """One NVML sample now (also called from the timing loop, so samples
        under load exist even when the sampler thread is starved)."""
        if self.nvml is None:
            return
        nv, handle, smax, bits = self.nvml
        try:
            sm = float(nv.nvmlDeviceGetClockInfo(handle, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(handle)
            self.samples.append((sm, smax, {k for k, b in bits.items() if r & b}))
        except Exception:
            pass

    def _nvml_loop(self):
        while not self.stop.is_set():
            self.poll()
            self.stop.wait(0.002)

    def __enter__(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            if vis and vis.split(",")[0].strip().isdigit():
                idx = int(vis.split(",")[self.device].strip())
            handle = nv.nvmlDeviceGetHandleByIndex(idx)
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            smax = float(nv.nvmlDeviceGetMaxClockInfo(handle, nv.NVML_CLOCK_SM))
            self.nvml = (nv, handle, smax, bits)
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            return
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for ln in out.splitlines():
                f = [x.strip() for x in ln.split(",")]
                if len(f) < 9:
                    continue
                try:
                    self.samples.append((float(f[1]), float(f[2]),
                                         {nm for nm, v in zip(self.NAMES, f[5:9])
                                          if v.lower() == "active"}))
                except ValueError:
                    continue

    def summary(self):
        sm = [x[0] for x in self.samples]
        smax = max((x[1] for x in self.samples), default=0.0)
        reasons = set().union(*[x[2] for x in self.samples]) if self.samples else set()
        load = [x for x in sm if x > 0.5 * (smax or 1)]
        return {"sm_mhz": float(np.median(load)) if load else (float(np.median(sm)) if sm else None),
                "sm_max_mhz": smax or None, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


def cpu_reference_time(cfg, j, sample_nnz, steps=1, warmup=1):
    """Times ftkref::epoch_plus (the unmodified reference, oracle/_ref) on this
    host's cores on a bounded sample of the workload; falls back to the C
    oracle port.  Data from datagen, model from ftkref::init_model: nothing
    of the engine package is loaded."""
    import datagen
    import oracle as O

    cores = os.cpu_count() or 1
    t = datagen.uniform_numpy(cfg["dims"], sample_nnz, cfg["seed"] + 100, cfg["lo"], cfg["hi"])
    tt = O.Tensor(t.dims, t.idx, t.vals)
    order = t.order
    sample = (f"{sample_nnz} nnz of the {cfg_name_of(cfg)} shape {list(cfg['dims'])}, J=R={j}, "
              f"{warmup} warm-up + {steps} measured epoch(s)")
    if O.REF is not None:
        R = O.REF
        scale = R.default_init_scale(float(np.mean(np.abs(t.vals))), order, j, [j] * order)
        m = R.init_model(t.dims, [j] * order, j, R.derive_seed(1, [77]), scale)
        _, secs = R.timed_epochs(tt, m, [R.derive_seed(1, [k + 1]) for k in range(warmup + steps)],
                                 workers=cores)
        dt = float(np.mean([f + c for f, c in secs[warmup:]]))
        return {"value": sample_nnz / dt, "unit": "nnz/s", "cores": cores,
                "kind": "reference", "sample": sample}
    # port: the plain-C restatement, one thread
    rng = np.random.default_rng(1)
    m = O.random_model(t.dims, [j] * order, j, 1, 0.3)
    p1 = rng.permutation(tt.nnz).astype(np.int64)
    t0 = time.perf_counter()
    O.COracle.factor_phase(tt, m, p1, 16, 1e-3, 1e-4)
    O.COracle.core_phase(tt, m, p1, 16, 1e-3, 1e-4)
    dt = time.perf_counter() - t0
    return {"value": sample_nnz / dt, "unit": "nnz/s", "cores": 1, "kind": "port",
            "sample": sample}


def dtype_of(args, order, j):
    """Operand types of the tensor-core sweeps (all accumulate in fp32)."""
    if args.precision != "tf32":
        return "f32" if args.precision == "fp32" else args.precision
    if order == 3 and j == 32 and args.core16 and not args.store_c and args.tc_ws:
        return "tf32+f16"  # factor: tf32 operands; core: fp16 copy of A
    return "tf32"


def cfg_name_of(cfg):
    import datagen

    for k, v in datagen.CONFIGS.items():
        if v["dims"] == cfg["dims"]:
            return k
    return "custom"


def run_reference(args):
    """The reference arm: ftkref::epoch_plus (unmodified reference sources,
    oracle/_ref) with workers = all host cores, on the SAME training tensor
    the engine arm times (datagen.workload; generated on the GPU for the
    1e8-scale configs, then handed to the reference as host COO), model from
    ftkref::init_model as the reference CLI does it (ftk.cpp:169-173).  At
    1e8 nonzeros an epoch takes ~35 s on 16 cores, so the arm times one
    warm-up and one measured epoch of the whole tensor whatever --steps /
    --warmup say (both reported); smaller configs honour them.  Imports
    nothing from the engine package."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    import datagen
    import oracle as O

    R = O.REF
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libftkref.so not built (needs /root/reference at build)"}))
        return
    t0 = time.perf_counter()
    cfg, j, tr, _ = datagen.workload(args.config, args.rank, "uniform", local)
    t_gen = time.perf_counter() - t0
    order = tr.order
    cores = os.cpu_count() or 1
    big = tr.nnz >= 10_000_000
    warm = min(args.warmup, 1) if big else args.warmup
    steps = 1 if big else args.steps
    scale = R.default_init_scale(float(np.mean(np.abs(tr.vals.astype(np.float64)))), order, j,
                                 [j] * order)
    m = R.init_model(tr.dims, [j] * order, j, R.derive_seed(1, [77]), scale)
    t1 = time.perf_counter()
    _, secs = R.timed_epochs(O.Tensor(tr.dims, tr.idx, tr.vals), m,
                             [R.derive_seed(1, [k + 1]) for k in range(warm + steps)],
                             workers=cores)
    meas = secs[warm:]
    dt = float(np.mean([f + c for f, c in meas]))
    value = tr.nnz / dt
    sample = (f"the whole training tensor ({tr.nnz} nnz, {args.config} shape "
              f"{list(cfg['dims'])}, J=R={j}), {warm} warm-up + {steps} measured epoch(s), "
              f"EpochStats.seconds_factor + seconds_core")
    line = {
        "impl": "reference",
        "metric": "SGD nonzeros/sec per epoch (factor+core) at J=R=32, 1-8 B200; test RMSE",
        "value": value, "unit": "nnz/s", "n_gpus": args.gpus, "steps": steps,
        "warmup": warm, "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (datagen.workload: the engine arm's tensor, uniform values)",
        "config": {"workload": args.config, "dims": list(cfg["dims"]), "nnz": tr.nnz,
                   "J": j, "R": j, "M": 16, "mode": "hogwild (workers = host cores)",
                   "fingerprint_train": datagen.fingerprint(tr)},
        "phases_ms": {"factor": float(np.mean([f for f, _ in meas])) * 1e3,
                      "core": float(np.mean([c for _, c in meas])) * 1e3},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "seconds": {"generate": t_gen, "epochs": time.perf_counter() - t1},
    }
    print(json.dumps(line), flush=True)


class SingleGpu:
    """Whole tensor on one session: one factor + one core sweep per epoch."""

    scaling = "weak"

    def __init__(self, eng, host, s, coo, ranks, j, a0, b0, world):
        self.eng, self.host, self.s, self.coo = eng, host, s, coo
        self.ranks, self.j, self.a0, self.b0, self.world = ranks, j, a0, b0, world
        self.parallelism = f"replica x{world}" if world > 1 else "1 GPU"
        self.local_nnz = coo.nnz
        self.job_nnz = coo.nnz * world  # independent replicas
        self.slot = 0

    def upload(self):
        self.s.upload_tensor(0, self.coo.dims, self.coo.idx, self.coo.vals)

    def upload_ptr(self, idx_ptr, val_ptr):
        self.s.upload_tensor_ptr(0, self.coo.dims, self.coo.nnz, idx_ptr, val_ptr)

    def upload_ptr_async(self, slot, idx_ptr, val_ptr):
        self.s.upload_tensor_ptr_async(slot, self.coo.dims, self.coo.nnz, idx_ptr, val_ptr)

    def upload_packed_async(self, slot, keys, val_ptr):
        lo, hi = keys
        self.s.upload_tensor_packed_ptr_async(slot, self.coo.dims, self.coo.nnz, lo.data_ptr(),
                                              None if hi is None else hi.data_ptr(), val_ptr)

    def host_arrays(self):
        return self.coo.idx, self.coo.vals

    def factor(self, es):
        self.s.factor_phase(self.slot, None, 16, 1e-3, 1e-4, self.eng.MODE_HOGWILD,
                            seed=self.host.derive_seed(es, [1]), timed=False)

    def core(self, es):
        self.s.core_phase(self.slot, None, 16, 1e-3, 1e-4, self.eng.MODE_HOGWILD,
                          seed=self.host.derive_seed(es, [2]), timed=False)

    def train_loss(self):
        out = self.s.eval(0, 1, 1e-4, 1e-4)
        return float(out[0] + out[2])

    def add_test(self, test):
        self.n_test = test.nnz
        self.s.upload_tensor(1, test.dims, test.idx, test.vals)

    def test_rmse_mae(self):
        """ftk::evaluate on the held-out set (evaluation.cpp:55-72)."""
        out = self.s.eval(1, 1, 0.0, 0.0)
        return float(np.sqrt(out[0] / self.n_test)), float(out[1] / self.n_test)


class Dsgd(SingleGpu):
    """DSGD strata over the ranks (paper_2404_10087_b200/dsgd.py): rank g
    holds mode-1 block g, sweeps one cell per stratum, ring-shifts the mode-2/3
    blocks over NCCL; the core phase all-reduces dB.  Total work is fixed."""

    scaling = "strong"

    def __init__(self, eng, host, s, coo, ranks, j, a0, b0, world, rank, schedule="strata",
                 tokens=1, runs=True):
        from paper_2404_10087_b200 import dsgd

        super().__init__(eng, host, s, coo, ranks, j, a0, b0, world)
        ring = schedule == "ring" and world > 1
        self.parallelism = (f"dsgd ring {world} ranks x {tokens * world} mode-3 blocks" if ring
                            else f"dsgd {world}x{world} strata" if world > 1 else "dsgd 1 cell")
        if runs:
            self.parallelism += ", cells in mode-3 runs"
        self.rank = rank
        self.layout = (dsgd.make_ring_layout(coo.dims, coo.idx, world, tokens) if ring
                       else dsgd.make_layout(coo.dims, coo.idx, world))
        self.idx, self.vals, self.off, _ = (dsgd.ring_cells if ring else dsgd.local_cells)(
            self.layout, coo.idx, coo.vals, rank, runs=runs)
        self.local_nnz = int(self.vals.shape[0])
        self.job_nnz = coo.nnz
        self.be = dsgd.EngineBackend(s, 0, self.idx, self.vals, self.off, coo.dims, coo.nnz,
                                     rank=rank, world=world, runs=runs)
        if ring:
            # peer descriptors around the ring (CUDA IPC handles), left neighbour mapped
            import torch.distributed as tdist

            blobs = [None] * world
            tdist.all_gather_object(blobs, s.ring_export())
            s.ring_connect(0, blobs[(rank - 1) % world])
            tdist.barrier()
        self.ring = ring
        self.tr = dsgd.DsgdTrainer(self.be, self.layout, rank,
                                   schedule="ring" if ring else "strata")

    def ring_ok(self):
        """One untimed ring factor phase; False on every rank if any rank's
        wait timed out (the caller then falls back to the strata)."""
        import torch
        import torch.distributed as tdist

        try:
            self.factor(self.host.derive_seed(3, [0]))
            bad = 1.0 if self.s.ring_status() else 0.0
        except Exception as e:  # noqa: BLE001
            print(f"bench: ring probe failed: {e}", file=sys.stderr)
            bad = 1.0
        bad = torch.tensor([bad], device=torch.device("cuda", torch.cuda.current_device()))
        tdist.all_reduce(bad, op=tdist.ReduceOp.MAX)
        return bad.item() == 0.0

    def upload(self):
        self.s.upload_tensor(0, self.coo.dims, self.idx, self.vals)
        self.s.set_cells(0, self.off)

    def upload_ptr(self, idx_ptr, val_ptr):
        self.s.upload_tensor_ptr(0, self.coo.dims, self.local_nnz, idx_ptr, val_ptr)
        self.s.set_cells(0, self.off)

    def host_arrays(self):
        return self.idx, self.vals

    def factor(self, es):
        self.tr.factor_phase(self.host.derive_seed(es, [1]))

    def core(self, es):
        self.tr.core_phase(es)

    def train_loss(self):
        self.tr.finalize()
        return float(self.tr.loss())

    def add_test(self, test):
        # after finalize() every rank holds the whole model: any share works
        self.n_test = test.nnz
        self.be.add_eval(np.ascontiguousarray(test.idx[self.rank::self.world]),
                         np.ascontiguousarray(test.vals[self.rank::self.world]), test.dims)

    def test_rmse_mae(self):
        return self.tr.rmse_mae(1)


def run_engine(args):
    import torch

    import datagen
    import paper_2404_10087_b200 as eng
    from paper_2404_10087_b200 import host

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    cfg, j, coo, test = datagen.workload(args.config, args.rank, "uniform", local)
    order = coo.order
    ranks = [j] * order
    s = eng.Session(local)
    prec = {"fp32": eng.PREC_FP32, "tf32": eng.PREC_TF32, "3xtf32": eng.PREC_3XTF32}[args.precision]
    s.set_option("precision", prec)
    s.set_option("eval", eng.EVAL_FAST)
    s.set_option("hog_update", args.hog_update)
    s.set_option("tc_ws", args.tc_ws)
    s.set_option("store_c", args.store_c)
    s.set_option("core16", args.core16)
    s.set_option("factor_warps", args.factor_warps)
    s.set_option("runs", args.runs)
    s.set_option("delta_decode", args.delta_decode)
    # the reference CLI's init (ftk.cpp:169-173): mean |x| over the training values
    scale = host.default_init_scale(float(np.mean(np.abs(coo.vals.astype(np.float64)))), order, j,
                                    ranks)
    a0, b0 = host.init_model(coo.dims, ranks, j, host.derive_seed(1, [77]), scale)
    s.upload_model(coo.dims, ranks, j, a0, b0)
    use_dsgd = (world > 1 or args.dsgd) and order == 3
    if use_dsgd:
        if world > 1:
            # NCCL id for the session's own communicator, shipped over the PG
            uid = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                uid.copy_(torch.frombuffer(bytearray(eng.Session.comm_unique_id()),
                                           dtype=torch.uint8))
            torch.distributed.broadcast(uid, 0)
            s.comm_init(bytes(uid.cpu().numpy().tobytes()), rank, world)
        sched = args.schedule if args.schedule != "auto" else ("strata" if world <= 2 else "ring")
        job = Dsgd(eng, host, s, coo, ranks, j, a0, b0, world, rank, sched, args.tokens,
                   args.cell_order == "runs")
        if job.ring and not job.ring_ok():
            print("bench: a DSGD ring wait timed out; falling back to the strata schedule",
                  file=sys.stderr)
            s.upload_model(coo.dims, ranks, j, a0, b0)
            job = Dsgd(eng, host, s, coo, ranks, j, a0, b0, world, rank, "strata", args.tokens,
                       args.cell_order == "runs")
    else:
        job = SingleGpu(eng, host, s, coo, ranks, j, a0, b0, world)
        job.upload()
    job.add_test(test)
    ext = torch.cuda.ExternalStream(s.stream_handle, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    for k in range(args.warmup):
        es = host.derive_seed(1, [k + 1])
        job.factor(es)
        job.core(es)
    loss0 = job.train_loss()
    test0 = job.test_rmse_mae()
    barrier()
    # per-phase events inside the timed region (same stream as the kernels)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    launches0 = s.get_option("launches")
    with ClockSampler(local) as clk:
        barrier()
        evs[0].record(ext)
        for k in range(args.steps):
            es = host.derive_seed(1, [args.warmup + k + 1])
            job.factor(es)
            evs[2 * k + 1].record(ext)
            job.core(es)
            evs[2 * k + 2].record(ext)
        while not evs[-1].query():  # clocks under load from this thread as well
            clk.poll()
            time.sleep(0.001)
        barrier()
    launches = s.get_option("launches") - launches0
    total_ms = evs[0].elapsed_time(evs[-1])
    kernels = kernel_names(s)
    f_ms = [evs[2 * k].elapsed_time(evs[2 * k + 1]) for k in range(args.steps)]
    c_ms = [evs[2 * k + 1].elapsed_time(evs[2 * k + 2]) for k in range(args.steps)]
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    loss1 = job.train_loss()
    test1 = job.test_rmse_mae()
    ms_step = total_ms / args.steps
    value = job.job_nnz / (ms_step * 1e-3)

    # roofline of the dominant kernel (algorithmic bytes) on
    # this rank's share of the nonzeros
    rec = 4 * order + 4
    f_bytes = job.local_nnz * (rec + 8 * sum(ranks))
    c_bytes = job.local_nnz * (rec + 4 * sum(ranks))
    f_avg, c_avg = float(np.mean(f_ms)), float(np.mean(c_ms))
    if f_avg >= c_avg:
        dom, dom_bytes, dom_ms = "factor", f_bytes, f_avg
    else:
        dom, dom_bytes, dom_ms = "core", c_bytes, c_avg
    peak, peak_kind = peaks()
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(TRAFFIC_PATH) as f:
            tr = json.load(f)
        key = f"{args.config}_j{j}_{args.precision}_{dom}"
        traffic = tr.get(key)
    except Exception:
        pass

    # The binding ceiling at L2-resident shapes: the factor
    # sweep's RED.v4 write-back alone on the same tile stream, measured live
    # (ftkcu_writeback_ceiling); its bytes = the sweep's algorithmic write-back
    # bytes (4 * sum J per nonzero).
    wb = None
    if order == 3 and all(x == 32 for x in ranks) and j == 32 and dom == "factor" \
            and type(job) is SingleGpu and args.hog_update:
        wb_ms = [s.writeback_ceiling(0, host.derive_seed(1, [k + 1])) for k in range(4)][1:]
        wb_bytes = job.local_nnz * 4 * sum(ranks)
        wb = {"ms": float(np.mean(wb_ms)), "bytes": wb_bytes}

    e2e = None
    if not args.no_e2e:
        e2e = time_e2e(job, a0, b0, args, torch, world, dev)

    # the same epochs at fp32-equivalent precision (3xtf32 split products on
    # the tensor cores), timed the same way after their own warm-up
    fp32_equiv = None
    if args.precision == "tf32" and not args.no_fp32_equiv and type(job) is SingleGpu:
        fp32_equiv = time_variant(job, s, eng, host, ext, torch, args, a0, b0,
                                  {"precision": eng.PREC_3XTF32}, barrier)
        fp32_equiv["value"] = job.job_nnz / (fp32_equiv["ms_per_step"] * 1e-3)
        s.set_option("precision", prec)

    rmse_ref = None
    if rank == 0 and world == 1 and not args.no_rmse_check:
        rmse_ref = rmse_vs_reference(args, cfg, j, coo, test, s, eng, host)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = min(args.cpu_sample, coo.nnz)
        cpu = cpu_reference_time(cfg, j, sample)

    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": "SGD nonzeros/sec per epoch (factor+core) at J=R=32, 1-8 B200; test RMSE",
            "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": job.scaling, "vs_baseline": None,
            "dtype": dtype_of(args, order, j),
            "data": "synthetic (uniform distinct tuples, values U[lo,hi], seeded)",
            "config": {"workload": args.config, "dims": list(cfg["dims"]), "nnz": coo.nnz,
                       "J": j, "R": j, "M": 16, "mode": "hogwild", "precision": args.precision,
                       "core_scheme": "storage" if args.store_c else "calculation",
                       "operands": {"factor": args.precision,
                                    "core": "f16 (RN copy of A, 10-bit mantissa)"
                                    if dtype_of(args, order, j) == "tf32+f16" else args.precision,
                                    "accumulate": "f32"},
                       "parallelism": job.parallelism, "nnz_per_rank": job.local_nnz,
                       "test_frac": cfg.get("test_frac", 0.014),
                       "l2": "no flush between steps: the COO tile stream (16 B/nnz per sweep) "
                             "is larger than L2; the factor rows stay L2-resident when they fit "
                             "(C2: 64 MB of the 126 MB L2; C3: 208 MB do not)"},
            "phases_ms": {"factor": f_avg, "core": c_avg},
            "train_loss_before_after": [loss0, loss1],
            "test_rmse_before_after": [test0[0], test1[0]],
            "test_mae_before_after": [test0[1], test1[1]],
            "test_nnz": test.nnz,
            "test_rmse_vs_reference": rmse_ref,
            "kernels": kernels,
            "value_fp32_equiv": None if fp32_equiv is None else fp32_equiv["value"],
            "fp32_equiv": fp32_equiv,
            "roofline": roofline_of(dom, dom_ms, dom_bytes, achieved, peak, peak_kind, traffic,
                                    wb, datagen.algorithmic_bytes_per_nnz(order, ranks),
                                    {"factor": f_avg, "core": c_avg},
                                    {"factor": f_bytes, "core": c_bytes,
                                     "core_rows": job.local_nnz * order},
                                    sum(int(d) * r * 4 for d, r in zip(coo.dims, ranks))),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    s.close()
    if world > 1:
        torch.distributed.destroy_process_group()


# TMA tile::gather4 row-rate ceiling measured on this pool's B200 (rows/s,
# profiles/r02_gather_rate.txt): the core sweep's binding limit.
GATHER_ROW_CEILING = 59.3e9

KERNEL_NAMES = {  # FTKCU_K_* (include/ftkcu.h) per sweep
    "factor": {1: "det_factor_kernel", 2: "ws_factor_kernel", 5: "wsf_factor_kernel",
               6: "wsg_factor_kernel", 7: "big_factor_kernel", 8: "tc_factor_kernel",
               9: "hog_factor_kernel", 10: "ws_factor3_kernel"},
    "core": {1: "det_core_kernel", 2: "ws_core_kernel", 3: "ws_core16_kernel",
             4: "ws_core_cc_kernel", 6: "wsg_core_kernel", 7: "big_core_kernel",
             8: "tc_core_kernel", 9: "hog_core_kernel"},
}


def kernel_names(s):
    return {"factor": KERNEL_NAMES["factor"].get(s.get_option("last_factor_kernel")),
            "core": KERNEL_NAMES["core"].get(s.get_option("last_core_kernel"))}


def time_variant(job, s, eng, host, ext, torch, args, a0, b0, opts, barrier):
    """W warm-up + K timed epochs from the initial model under session
    options `opts` (CUDA events on the session stream)."""
    for k, v in opts.items():
        s.set_option(k, v)
    s.upload_model(job.coo.dims, job.ranks, job.j, a0, b0)
    for k in range(args.warmup):
        es = host.derive_seed(1, [k + 1])
        job.factor(es)
        job.core(es)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    barrier()
    evs[0].record(ext)
    for k in range(args.steps):
        es = host.derive_seed(1, [args.warmup + k + 1])
        job.factor(es)
        evs[2 * k + 1].record(ext)
        job.core(es)
        evs[2 * k + 2].record(ext)
    barrier()
    f = [evs[2 * k].elapsed_time(evs[2 * k + 1]) for k in range(args.steps)]
    c = [evs[2 * k + 1].elapsed_time(evs[2 * k + 2]) for k in range(args.steps)]
    return {"options": {k: int(v) for k, v in opts.items()},
            "ms_per_step": evs[0].elapsed_time(evs[-1]) / args.steps,
            "phases_ms": {"factor": float(np.mean(f)), "core": float(np.mean(c))},
            "kernels": kernel_names(s),
            "dtype": "3xtf32 (fp32-equivalent split products, fp32 accumulate)"
            if opts.get("precision") == eng.PREC_3XTF32 else None}


L2_RESIDENT_MAX = 96e6  # factor rows up to here stay in the 126 MB L2 (C2: 64 MB; C3: 208 MB)


def roofline_of(dom, dom_ms, dom_bytes, achieved, peak, peak_kind, traffic, wb, bpn, ms, nbytes,
                a_bytes=0):
    """The dominant kernel against the ceiling that binds it.  At the
    Netflix shape the factor rows are L2-resident (ncu: DRAM ~4 % busy), so
    algorithmic bytes over HBM peak exceeds 1 and says nothing; the binding
    ceiling is the L2 atomic (RED) rate of the sweep's own write-back,
    measured live on the same tile stream.  When the rows do not fit L2
    (Yahoo: 208 MB) the sweep is HBM-bound: its fraction is the ncu DRAM
    bytes per launch (`traffic`) over the live kernel time against the
    measured HBM peak (algorithmic bytes would count the L2 hits of the
    small modes).  The algorithmic HBM view stays alongside."""
    hbm = {"achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "peak_source": peak_kind, "algorithmic_bytes_per_launch": dom_bytes,
           "bytes_per_nnz_epoch": bpn,
           "per_kernel_frac": {k: nbytes[k] / (ms[k] * 1e-3) / 1e9 / peak for k in ms}}
    if a_bytes > L2_RESIDENT_MAX and dom_ms > 0 and traffic:
        dram = traffic / (dom_ms * 1e-3) / 1e9
        return {"bound": "hbm", "kernel": dom, "achieved": dram, "peak": peak, "unit": "GB/s",
                "frac": dram / peak, "peak_source": peak_kind,
                "achieved_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                   "(profiles/ncu_traffic.json) / live kernel time",
                "factor_rows_bytes": a_bytes, "traffic": traffic, "algorithmic": hbm}
    if wb is None or dom_ms <= 0:
        out = {"bound": "hbm", "kernel": dom}
        out.update(hbm)
        out["traffic"] = traffic
        return out
    ach = wb["bytes"] / (dom_ms * 1e-3) / 1e9
    ceil = wb["bytes"] / (wb["ms"] * 1e-3) / 1e9
    kernels = {"factor": {"bound": "l2_red", "achieved_GBs": ach, "peak_GBs": ceil,
                          "frac": ach / ceil}}
    if "core" in ms and ms["core"] > 0 and nbytes.get("core_rows"):
        rows_s = nbytes["core_rows"] / (ms["core"] * 1e-3)
        kernels["core"] = {
            # no single resource is saturated (ncu, profiles/r02_final_netflix_ws_core16_*:
            # tensor pipe 30%, L1 44%, L2 20%, DRAM 5%; stalls on TMEM / L1TEX loads);
            # the isolated TMA gather microbenchmark is exceeded, so it is no ceiling
            "bound": "latency (no unit saturated)", "achieved_rows_per_s": rows_s,
            "isolated_gather4_rows_per_s": GATHER_ROW_CEILING,
            "gather_source": "profiles/r02_gather_rate.txt, r02_gather_rate_mix.txt "
                             "(scripts/microtests/gather_rate.cu)",
            "rows_note": "3 gathered rows (one per mode) per nonzero"}
    return {"bound": "l2_red", "kernel": dom, "achieved": ach, "peak": ceil, "unit": "GB/s",
            "frac": ach / ceil, "kernels": kernels,
            "peak_source": ("measured live: ftkcu_writeback_ceiling, the sweep's RED.v4 "
                            "write-back alone on the same tile stream "
                            f"({wb['ms']:.3f} ms for {wb['bytes']} B)"),
            "algorithmic_bytes_per_launch": wb["bytes"],
            "bytes_note": "write-back bytes: 4 * sum(J) per nonzero (three 128-B row updates)",
            "traffic": traffic, "hbm": hbm}


TRAJ_PATH = os.path.join(ROOT, "tests", "golden", "c2_trajectory.json")


def reference_worker_spread():
    """How far the reference's own uniform-data trajectory moves between
    workers = 1 and workers = 16 (tests/golden/c2_workers_spread.json,
    oracle/ref_workers_spread.py: ftkref::train on a statistically equivalent
    C2 tensor) -- the scale against which an asynchronous engine's uniform
    RMSE delta reads."""
    path = os.path.join(ROOT, "tests", "golden", "c2_workers_spread.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        sp = json.load(f)
    if "1" not in sp or "16" not in sp:
        return None
    w1, w16 = sp["1"]["rmse"], sp["16"]["rmse"]
    return {"workers_1": w1, "workers_16": w16,
            "max_abs_delta": max(abs(a - b) for a, b in zip(w1, w16)),
            "tensor": "datagen cpu stream (statistically equivalent, not the bench bytes)"}


def rmse_vs_reference(args, cfg, j, coo, test, s, eng, host):
    """North-star accuracy at the benchmarked configuration: from the
    reference CLI's initial model, E Hogwild epochs of the engine (the same
    kernels and precision as the timed epochs) with the test RMSE after each,
    against ftkref::train's trajectory on the identical tensors
    (tests/golden/c2_trajectory.json, oracle/gen_c2_trajectory.py, run on the
    GPU box's host cores).  For the uniform benchmark data and for planted
    J = R = 32 values on the same tuples (whose RMSE moves).

    On uniform (unlearnable) values the RMSE after an epoch is a noise floor
    that rises with asynchrony: the full grid keeps ~57K nonzeros in flight
    (148 CTAs x 3 tiles x 128), ~26 per row of the 2182-row mode, whose
    summed stale steps act as a larger step.  The `parity` variant (window =
    3: a row slot is freed only after its tile's write-back, so at most 3
    tiles per CTA are between read and write; 74 CTAs) brings the floor
    within 1e-3 of the reference's at 2.1x the epoch time (the grid cap alone
    needs 37 CTAs, 3.7x); reported with its epoch time, not the headline."""
    import datagen

    if not os.path.exists(TRAJ_PATH):
        return None
    with open(TRAJ_PATH) as f:
        fx = json.load(f)
    out = {}
    for kind, ref in sorted(fx.items()):
        if ref["workload"] != args.config or ref["J"] != j:
            continue
        if kind == "uniform":
            tr, te = coo, test
        else:
            _, _, tr, te = datagen.workload(args.config, args.rank, kind, 0)
        fp = datagen.fingerprint(tr)
        order = tr.order
        scale = host.default_init_scale(float(np.mean(np.abs(tr.vals.astype(np.float64)))),
                                        order, j, [j] * order)
        a, b = host.init_model(tr.dims, [j] * order, j, host.derive_seed(1, [77]), scale)
        s.upload_tensor(4, tr.dims, tr.idx, tr.vals)
        s.upload_tensor(5, te.dims, te.idx, te.vals)
        want = [ref["rmse_init"]] + ref["rmse"]
        variants = [("default", {})]
        if kind == "uniform":
            variants.append(("parity (window 3, 74 CTAs)", {"window": 3, "max_ctas": 74}))
            variants.append(("last-mode runs", {"runs": 1}))
            # the reference's sampler redraws every nonzero's position each
            # epoch (sparse_tensor.cpp:271-282); the engine shuffles once per
            # upload and permutes whole tiles per epoch.  This variant rebuilds
            # the stream with a fresh seed before every epoch (the rebuild is
            # not in its epoch_ms, which times the sweep kernels)
            variants.append(("reshuffled every epoch", {"reshuffle": 1}))
        res = {}
        for name, opts in variants:
            reshuffle = bool(opts.get("reshuffle"))
            opts_set = {k: v for k, v in opts.items() if k != "reshuffle"}
            if reshuffle:
                opts_set["shuffle_seed"] = s.get_option("shuffle_seed")
            prev = {k: s.get_option(k) for k in opts_set}
            for k, v in opts_set.items():
                s.set_option(k, v)
            s.upload_model(tr.dims, [j] * order, j, a, b)
            ev = s.eval(5, 1, 0.0, 0.0)
            rm = [float(np.sqrt(ev[0] / te.nnz))]
            ep_ms = []
            for e in range(len(ref["rmse"])):
                es = host.derive_seed(1, [e + 1])
                if reshuffle:
                    s.set_option("shuffle_seed", int(host.derive_seed(es, [3]) & 0x7fffffffffffffff))
                f_ms = s.factor_phase(4, None, 16, ref["lr_a"], ref["reg_a"], eng.MODE_HOGWILD,
                                      seed=host.derive_seed(es, [1]), timed=True)
                c_ms = s.core_phase(4, None, 16, ref["lr_b"], ref["reg_b"], eng.MODE_HOGWILD,
                                    seed=host.derive_seed(es, [2]), timed=True)
                ep_ms.append(float(f_ms) + float(c_ms if np.isscalar(c_ms) else c_ms[0]))
                ev = s.eval(5, 1, 0.0, 0.0)
                rm.append(float(np.sqrt(ev[0] / te.nnz)))
            for k, v in prev.items():
                s.set_option(k, v)
            dev = [abs(x - y) for x, y in zip(rm, want)]
            res[name] = {"engine": rm, "max_abs_delta": max(dev),
                         "within_1e-3": bool(max(dev) <= 1e-3), "options": opts,
                         "kernels": kernel_names(s),
                         # device ms per epoch of these (untimed-region) epochs and the
                         # throughput they imply: the price of the variant
                         "epoch_ms": float(np.median(ep_ms)),
                         "nnz_per_s": tr.nnz / (float(np.median(ep_ms)) * 1e-3)}
        out[kind] = dict(res["default"], reference=want, same_tensor=fp == ref["fingerprint_train"],
                         reference_workers=ref["workers"])
        spread = reference_worker_spread() if kind == "uniform" else None
        if spread:
            out[kind]["reference_worker_spread"] = spread
        if len(res) > 1:
            out[kind]["variants"] = {k: v for k, v in res.items() if k != "default"}
        s.release_tensor(4)
        s.release_tensor(5)
    return out or None


# e2e tensor slots (slot 0: the device-timed tensor; 4 / 5: the RMSE check)
E2E_SLOTS = (2, 3, 6)


def time_e2e(job, a0, b0, args, torch, world, dev):
    """Same epochs through the C-ABI from pinned host buffers, host<->device
    copies of every step's inputs (this rank's COO share + model) and result
    (model) inside the timed region; max over ranks."""
    from paper_2404_10087_b200 import host

    idx, vals = job.host_arrays()
    pipelined = type(job) is SingleGpu and not args.e2e_sync
    # packed-key COO on the link (ftkcu_pack_keys, built once like a file
    # format; 12 instead of 16 bytes per nonzero), where the index widths fit
    keys = None
    delta = None
    if pipelined and args.e2e_keys == "delta":
        # delta-coded COO (ftkcu_pack_delta: sorted mixed-radix keys, chunked
        # deltas; built once like a file format, untimed): the values travel
        # in the sorted order
        try:
            de, rs, vo, w = job.s.pack_delta(job.coo.dims, idx, vals)
            delta = (torch.from_numpy(de).pin_memory(), torch.from_numpy(rs.view(np.int64))
                     .pin_memory(), w)
            vals = vo
        except Exception:
            delta = None
    if pipelined and args.e2e_keys == "packed":
        try:
            keys = job.s.pack_keys(job.coo.dims, idx)
        except Exception:
            keys = None
    if delta is not None:
        de_h, rs_h, width = delta
        key_bytes = de_h.numel() + rs_h.numel() * 8

        def upload_async(sl, _idx_ptr, vptr):
            job.s.upload_tensor_delta_ptr_async(sl, job.coo.dims, job.coo.nnz, de_h.data_ptr(),
                                                width, rs_h.data_ptr(), vptr)
        idx_h = de_h
    elif keys is not None:
        lo, hi = keys
        key_h = (torch.from_numpy(lo.view(np.int32)).pin_memory(),
                 None if hi is None else torch.from_numpy(hi.view(np.int16 if hi.itemsize == 2
                                                                  else np.int32)).pin_memory())
        key_bytes = lo.nbytes + (0 if hi is None else hi.nbytes)

        def upload_async(sl, _idx_ptr, vptr):
            job.upload_packed_async(sl, key_h, vptr)
        idx_h = key_h[0]
    else:
        idx_h = torch.from_numpy(np.ascontiguousarray(idx)).pin_memory()
        key_bytes = idx_h.numel() * idx_h.element_size()
        upload_async = job.upload_ptr_async
    val_h = torch.from_numpy(np.ascontiguousarray(vals)).pin_memory()
    a_h = [torch.from_numpy(x.copy()).pin_memory() for x in a0]
    b_h = [torch.from_numpy(x.copy()).pin_memory() for x in b0]
    a_np = [x.numpy() for x in a_h]
    b_np = [x.numpy() for x in b_h]
    # Single GPU: tensor slots E2E_SLOTS in rotation, step k + 1's COO copy
    # (ftkcu_tensor_upload_*_async, copy stream) overlapping step k's epoch.
    # Three slots, not two: with two, step k+1's copy had to wait for epoch
    # k-1 (the last reader of its slot), so the link idled between the end of
    # copy k and the end of epoch k-1 (5.8 ms of an 18.5 ms step in the
    # FTK_E2E_TRACE timeline) and the last parts of the upload were decoded
    # after the core sweep instead of beside the factor sweep.
    nsl = len(E2E_SLOTS)
    steps = max(1, args.steps if pipelined else min(args.steps, 3))
    h2d = key_bytes + vals.nbytes + (0 if pipelined else sum(x.nbytes for x in a_np + b_np))
    d2h = sum(x.nbytes for x in a_np + b_np)
    s = job.s
    if pipelined:
        # untimed: allocate both slots' device buffers (COO, staging, tile
        # stream) once; every timed step still copies its whole COO again
        for sl in E2E_SLOTS:
            upload_async(sl, idx_h.data_ptr(), val_h.data_ptr())
            job.slot = sl
            job.factor(host.derive_seed(5, [sl]))
        s.model_copy_async(False, a_np, b_np)  # read-back snapshot buffer
        s.sync()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    trace = os.environ.get("FTK_E2E_TRACE") == "1"  # host timeline (diagnostics)
    t0 = time.perf_counter()

    ext = torch.cuda.ExternalStream(s.stream_handle, device=dev)
    tev = []

    def mark(what):
        if trace:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(ext)
            tev.append((what, ev))
            print(f"e2e {(time.perf_counter() - t0) * 1e3:8.2f} ms {what}", file=sys.stderr)

    cps = torch.cuda.ExternalStream(s.get_option("copy_stream"), device=dev) if trace else None

    dcs = torch.cuda.ExternalStream(s.get_option("dec_stream"), device=dev) if trace else None

    def mark_copy(what):
        if trace:
            for st, w in ((cps, what), (dcs, what.replace("copied", "decoded"))):
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(st)
                tev.append((w, ev))

    mark("start")
    if pipelined:
        upload_async(E2E_SLOTS[0], idx_h.data_ptr(), val_h.data_ptr())
        mark_copy("[copy] upload 0 copied")
    for k in range(steps):
        if not pipelined:
            job.upload_ptr(idx_h.data_ptr(), val_h.data_ptr())
            s.upload_model(job.coo.dims, job.ranks, job.j, a_np, b_np)
        # pipelined: the model stays resident across steps (it is the
        # training state, not an input); each step's result is read back
        mark(f"step {k} model uploaded")
        if pipelined and k + 1 < steps:
            # step k+1's COO, enqueued before this step's epoch: the copy
            # engine streams it right behind step k's copy (it waits only for
            # step k+1-nsl, the last epoch that read its slot), so the link
            # stays busy while step k computes
            upload_async(E2E_SLOTS[(k + 1) % nsl], idx_h.data_ptr(), val_h.data_ptr())
            mark("next upload enqueued")
            mark_copy(f"[copy] upload {k + 1} copied")
        if pipelined:
            job.slot = E2E_SLOTS[k % nsl]
        es = host.derive_seed(7, [k + 1])
        job.factor(es)
        mark("factor enqueued")
        job.core(es)
        mark("core enqueued")
        if pipelined:
            s.model_copy_async(False, a_np, b_np)
        else:
            s.download_model(a_np, b_np)
        mark("model downloaded")
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    for what, ev in sorted(tev, key=lambda x: tev[0][1].elapsed_time(x[1])):
        print(f"e2e gpu {tev[0][1].elapsed_time(ev):8.2f} ms {what}", file=sys.stderr)
    if pipelined:
        job.slot = 0
        for sl in E2E_SLOTS:
            s.release_tensor(sl)
    if world > 1:
        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": job.job_nnz / dt, "unit": "nnz/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": dt * 1e3, "steps": steps,
            "keys": (f"delta-coded ({key_bytes / job.coo.nnz:.2f} B/nnz: {width}-byte deltas of "
                     f"sorted mixed-radix keys + a restart key per 4096, ftkcu_pack_delta, built "
                     f"once like a file format; {(key_bytes + vals.nbytes) / job.coo.nnz:.2f} "
                     f"B/nnz with the values)") if delta is not None else
                    (f"packed ({key_bytes / job.coo.nnz:.0f} B/nnz, ftkcu_pack_keys; "
                     f"{(key_bytes + vals.nbytes) / job.coo.nnz:.0f} B/nnz with the values)")
                    if keys is not None else "int32 per mode (16 B/nnz with values)",
            "path": (("ftkcu_tensor_upload_delta_async" if delta is not None else
                      "ftkcu_tensor_upload_packed_async" if keys is not None else
                      "ftkcu_tensor_upload_async") + f" into {nsl} rotating slots (step k+1's COO "
                     "copy overlaps step k's epoch)" if pipelined else "ftkcu_tensor_upload")
                    + (" + factor/core phases + the model read back every step "
                       "(ftkcu_model_copy_async; the model stays resident)" if pipelined else
                       " + ftkcu_model_upload + factor/core phases + ftkcu_model_download")
                    + ", pinned host buffers (per rank, max over ranks)"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_engine(args)


if __name__ == "__main__":
    main()
