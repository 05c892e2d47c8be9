#!/usr/bin/env python
"""Benchmark of the partial-fraction exp(A)V hot path on B200 (BASELINE.json metric:
"exp(A)V evals/sec at 1/2/4/8 B200; % of FP64-tensor or HBM roofline").

Default workload = BASELINE configs[3] (C4), the largest single-GPU config and the one whose
text carries the metric's "1/2/4/8 GPUs": one dense complex Hermitian A, d = 4096, spectrum
U[-500, 0], the full exp(A) (V = I, 4096 RHS), n = 24 (12 conjugate pole pairs), one blocked
LU per shift.  One eval (= one step) = the whole 4096 x 4096 result.  --workload C1/C2/C3/C5
selects the other configs.  Inputs are seeded synthetic data with the reference recipes
(paper_2306_16778_b200/workloads.py); there is no dataset.

Multi-GPU (torchrun, one process per GPU), total work fixed as N grows ("scaling":
"strong"), --shard selects how it is split:
  pole   the n/2 pole pairs in contiguous ascending blocks; each rank factors and solves
         its own shifts and the partial sums meet in ONE NCCL reduce to rank 0 (the
         north-star mechanism; every config);
  rows   C2 only: each rank owns a contiguous block of the tridiagonal's row chunks
         (pfx_expm_tridiag_shard); the two chunk scans exchange one small all-gather each
         and every output row is final on its rank (no reduction of the 134 MB result);
  batch  C3 only: each rank solves its block of the 512 matrices (no collective);
  auto   rows for C2, batch for C3, pole otherwise (default: pole on every config).

Timing: W warm-up steps, then K steps between barrier + synchronize, CUDA events on
the launching stream, max over ranks; library profiling is off in the timed region (a
separate pass with per-launch CUDA events produces the kernel breakdown and the
dominant-kernel roofline).  L2 policy per config (config.l2): C2-C5 inputs exceed the
126 MB L2, so no flush; C1 (256 KB of inputs) writes a 256 MB buffer before every step and
times each step with its own event pair recorded after the flush (the K step durations are
summed; the flush sits between timed iterations).

`--impl reference` times the reference's own CPU implementation of the same workload on the
host cores (oracle/cpu_timer.py): the unmodified reference package from baseline/_ref through
its public API for the dense configs (matexp_action / matexp_full), the oracle restatement
(zgtsv / zgbsv per pole pair, 2 Re(a y), ascending reduction) for the structured ones, which
the dense-only reference cannot express.  BLAS threads are exported before numpy loads, the
inputs are built outside the timer, every step is one bounded sample of the workload, and the
value is the median step after the warm-up (reference bench.py:196-205).  The thread setting
is the best of BASELINE.md §3's three, recorded on the pod by `--cpu-calibrate`
(profiles/cpu_settings.json).  The same timer gives the GPU arm's `cpu_baseline`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "exp(A)V evals/sec"
UNIT = "evals/s"

# Algorithmic work per eval (complex counting: 8 real flops per complex FMA)
ALG_FLOPS = {
    "C1": 8.0 * (8.0 / 3.0 * 128**3 + 8.0 * 128**2),
    "C2": 12.0 * (1 << 20) * (12 + 16 * 22),
    "C3": 10.0 * (8.0 / 3.0 * 256**3 + 2 * 8.0 * 256**2),  # per matrix (one eval = one matrix)
    "C4": 12.0 * (8.0 / 3.0 + 16.0 / 3.0) * 4096**3,
    "C5": 8.0 * (8.0 * 262144 * 512 * 512 + 8.0 * 262144 * 1024 * 8),
}
ALG_BYTES = {
    "C1": 1.33e5,
    "C2": 8.0 * (1 << 20) * (2 + 2 * 16),
    "C3": 5.40e8 / 512,
    "C4": 5.37e8,
    "C5": 8.0 * 2 * 513 * 262144 * 16,
}
# Per-launch hardware counters of the dominant kernel from the round's ncu pass over the same
# bench command (tools/ncu_summary.py -> profiles/ncu_summary.json): mean dram__bytes_read.sum +
# dram__bytes_write.sum per launch, duration-weighted DMMA / FP64 pipe utilisation.
def load_ncu_summary():
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return {}
DOMINANT = {"C1": "dense_batched_kernel", "C2": "tri_sweep", "C3": "dense_batched_kernel", "C4": "zgemm", "C5": "zgemm"}


def load_peaks():
    peaks = {"hbm_gbs": 6488.0, "fp64_tflops": 36.9, "fp64_source": "profiles/fp64_peak_r01.txt (DMMA m8n8k4, measured)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            m = json.load(fh)
        peaks["hbm_gbs"] = float(m.get("hbm_gbs", peaks["hbm_gbs"]))
        if "fp64_tflops" in m:
            peaks["fp64_tflops"] = float(m["fp64_tflops"])
            peaks["fp64_source"] = "MEASURED_PEAKS.json"
    return peaks


# ---- clocks sampling -------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms around the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        # nvidia-smi's start-up (driver attach, ~0.1-0.3 s of host work) must not overlap the
        # timed region: return once it is in its sampling loop (first line out)
        t0 = time.perf_counter()
        while not self.lines and time.perf_counter() - t0 < 3.0 and self.proc.poll() is None:
            time.sleep(0.005)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


# ---- workloads -------------------------------------------------------------------

class Workload:
    """Inputs resident on the device + a step function calling the native library."""

    def __init__(self, name, torch, dev, pairs_lo, pairs_hi, batch_range=None, col_tasks=None, c1_batch=1):
        from paper_2306_16778_b200 import workloads as W
        from paper_2306_16778_b200.roots import default_table

        self.name = name
        self.torch = torch
        self.dev = dev
        if name == "C2":
            n = W.C2["n"]
            d, o = W.c2_matrix()
            V = W.c2_rhs()
            self.host = dict(diag=d, off=o, V=V)
            self.h2d = d.nbytes + o.nbytes + V.nbytes
            self.d2h = V.nbytes
            self.evals_per_step = 1.0
        elif name == "C1":
            n = W.C1["n"]
            A, v, _ = W.c1_inputs()
            if c1_batch > 1:
                # throughput mode: c1_batch independent C1 problems (trials 0..B-1 of the same
                # recipe) in one call, as the CPU arm runs one problem per process at a time
                A = np.stack([W.random_real_symmetric(W.C1["d"], W.C1["lo"], W.C1["hi"], 0, t)[0]
                              for t in range(c1_batch)])
                v = np.stack([W.unit_vector(W.C1["d"], 0, t) for t in range(c1_batch)])
            self.host = dict(A=A, V=v)
            self.h2d = A.nbytes + v.nbytes
            self.d2h = v.nbytes
            self.evals_per_step = float(c1_batch)
        elif name == "C3":
            n = W.C3["n"]
            A, V = W.c3_batch()
            self.host = dict(A=A, V=V)
            self.h2d = A.nbytes + V.nbytes
            self.d2h = V.nbytes * 2
            self.evals_per_step = float(W.C3["batch"])
        elif name == "C4":
            n = W.C4["n"]
            A, _ = W.c4_matrix()
            self.host = dict(A=A)
            self.h2d = A.nbytes
            self.d2h = A.nbytes
            self.evals_per_step = 1.0
        elif name == "C5":
            n = W.C5["n"]
            band = W.c5_band()
            V = W.c5_rhs()
            self.host = dict(band=band, V=V)
            self.h2d = band.nbytes + V.nbytes
            self.d2h = V.nbytes
            self.evals_per_step = 1.0
        else:
            raise SystemExit(f"unknown workload {name}")
        if batch_range is not None:  # batch sharding (C3): this rank's matrices only
            b0, b1 = batch_range
            self.host = {k: v[b0:b1] for k, v in self.host.items()}
        self.n = n
        t2, c2 = default_table(n).interleaved()
        self.theta2 = np.ascontiguousarray(t2[2 * pairs_lo: 2 * pairs_hi])
        self.coef2 = np.ascontiguousarray(c2[2 * pairs_lo: 2 * pairs_hi])
        # C4 at N > 1 with leftover pairs: this rank's (pair, c0, c1) tasks (sharding.colsplit_plan)
        self.col_ranges = None
        if col_tasks is not None:
            idx = [k for k, _, _ in col_tasks]
            self.theta2 = np.ascontiguousarray(np.concatenate([t2[2 * k: 2 * k + 2] for k in idx]))
            self.coef2 = np.ascontiguousarray(np.concatenate([c2[2 * k: 2 * k + 2] for k in idx]))
            self.col_ranges = np.array([[a, b] for _, a, b in col_tasks], dtype=np.int64)
        self.dev_in = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in self.host.items()}
        self.out = None
        self.flush = None
        if name == "C1":
            self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        # pinned host copies (inputs and result) for the end-to-end number
        self.pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in self.host.items()}
        out_elems = {"C2": 16 << 20, "C1": 128 * c1_batch, "C3": 512 * 256 * 2, "C4": 4096 * 4096 * 2, "C5": 262144 * 8}[name]
        self.pinned_out = torch.empty(out_elems, dtype=torch.float64).pin_memory()

    def step(self, stream):
        from paper_2306_16778_b200 import _native

        di = self.dev_in
        if self.name == "C2":
            self.out = _native.expm_tridiag_device(di["diag"], di["off"], di["V"], self.theta2, self.coef2, 0.0,
                                                   out=self.out, stream=stream)
        elif self.name in ("C1", "C3"):
            self.out = _native.expm_dense_device(di["A"], di["V"], self.theta2, self.coef2, 0.0, stream=stream)
        elif self.name == "C4" and self.col_ranges is not None:
            self.out = _native.expm_dense_cols_device(di["A"], self.theta2, self.coef2, self.col_ranges, 0.0,
                                                      out=self.out, stream=stream)
        elif self.name == "C4":
            self.out = _native.expm_dense_device(di["A"], None, self.theta2, self.coef2, 0.0, out=self.out,
                                                 stream=stream)
        elif self.name == "C5":
            self.out = _native.expm_banded_device(di["band"], di["V"], self.theta2, self.coef2, 0.0, out=self.out,
                                                  stream=stream)
        return self.out

    def step_host(self):
        """Same computation through the C-ABI with HOST buffers (PFX_MEM_HOST): H2D + compute + D2H."""
        from paper_2306_16778_b200 import _native

        p = {k: v.numpy() for k, v in self.pinned.items()}
        o = self.pinned_out.numpy()
        if self.name == "C2":
            return _native.expm_tridiag_host(p["diag"], p["off"], p["V"], self.theta2, self.coef2, 0.0, out=o)
        if self.name == "C1":
            return _native.expm_dense_host(p["A"], p["V"], self.theta2, self.coef2, 0.0, out=o)
        if self.name in ("C3", "C4"):
            oc = o.view(np.complex128)
            return _native.expm_dense_host(p["A"], p.get("V"), self.theta2, self.coef2, 0.0, out=oc)
        return _native.expm_banded_host(p["band"], p["V"], self.theta2, self.coef2, 0.0, out=o)


# ---- CPU baseline (the reference on the host cores) ---------------------------------

# BASELINE.md §3 thread settings: (processes, BLAS threads per process)
def cpu_settings(cores):
    return {"S1": (1, 1), "S2": (cores, 1), "S3": (1, cores)}


CPU_SETTINGS_FILE = os.path.join(ROOT, "profiles", "cpu_settings.json")
# survey winners, used until a calibration on the pod is recorded
CPU_DEFAULT_SETTING = {"C1": "S1", "C2": "S2", "C3": "S2", "C4": "S3", "C5": "S2"}


def cpu_best_setting(name):
    if os.path.exists(CPU_SETTINGS_FILE):
        with open(CPU_SETTINGS_FILE) as fh:
            rec = json.load(fh)
        if name in rec and "best" in rec[name]:
            return rec[name]["best"]
    return CPU_DEFAULT_SETTING[name]


def run_cpu(name, cores, setting, steps, warmup):
    """One oracle.cpu_timer subprocess (BLAS threads exported before numpy loads, inputs built
    once per process outside the timer, median of `steps` after `warmup`).  Returns its dict."""
    procs, blas = cpu_settings(cores)[setting]
    cmd = [sys.executable, "-m", "oracle.cpu_timer", "--workload", name, "--procs", str(procs), "--blas", str(blas),
           "--steps", str(steps), "--warmup", str(warmup)]
    env = dict(os.environ, OPENBLAS_NUM_THREADS=str(blas), OMP_NUM_THREADS=str(blas), MKL_NUM_THREADS=str(blas))
    env.pop("CUDA_VISIBLE_DEVICES", None)
    res = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"cpu_timer failed: {res.stderr[-2000:]}")
    out = json.loads(res.stdout.strip().splitlines()[-1])
    out["setting"] = setting
    return out


def cpu_calibrate(name, cores, steps=5, warmup=1):
    """Times all three settings (median of `steps` after `warmup` each) and records the best."""
    rec = {}
    if os.path.exists(CPU_SETTINGS_FILE):
        with open(CPU_SETTINGS_FILE) as fh:
            rec = json.load(fh)
    res = {s: run_cpu(name, cores, s, steps, warmup) for s in cpu_settings(cores)}
    best = max(res, key=lambda s: res[s]["value"])
    rec[name] = {"best": best, "nproc": cores, "cpu": _cpu_model(),
                 "settings": {s: {k: r[k] for k in ("value", "median_step_s", "procs", "blas_threads", "kind",
                                                     "sample", "blas")} for s, r in res.items()}}
    os.makedirs(os.path.dirname(CPU_SETTINGS_FILE), exist_ok=True)
    with open(CPU_SETTINGS_FILE, "w") as fh:
        json.dump(rec, fh, indent=1)
    return rec[name]


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_entry(r):
    return {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
            "sample": r["sample"] + f"; median of {r['steps']} after {r['warmup']} warm-up (setting {r['setting']})",
            "setting": r["setting"], "median_step_s": r["median_step_s"], "blas": r.get("blas"),
            "nproc": r.get("nproc"), "cpu": _cpu_model()}


def config_dict(name, world, shard):
    """The `config` object both arms print (identical for the same workload and N)."""
    desc = dict(WORKLOAD_DESC[name])
    desc["parallelism"] = {
        "pole": f"pole-shard x{world}" + (" + 1 NCCL reduce" if world > 1 else ""),
        "rows": f"row-shard x{world} + 2 small all-gathers (scan aggregates); output rows stay on their rank",
        "batch": f"batch-shard x{world} (no collective)"}[shard]
    return desc


WORKLOAD_DESC = {
    "C1": {"workload": "C1: dense real symmetric d=128, spectrum U[-50,0], exp(A)v, n=16", "d": 128, "n": 16,
           "l2": "256 MB L2 flush before every step, between the per-step CUDA event pairs"},
    "C2": {"workload": "C2: tridiagonal 1-D Dirichlet Laplacian, N=2^20, spectrum (-100,0), 16 RHS, n=24",
           "N": 1 << 20, "nrhs": 16, "n": 24,
           "l2": "inputs (144 MB) + output (128 MB) exceed L2 (126 MB); no flush"},
    "C3": {"workload": "C3: 512 dense complex Hermitian d=256, spectrum U[-200,0], exp(A)v, n=20",
           "batch": 512, "d": 256, "n": 20, "l2": "inputs 537 MB exceed L2; no flush"},
    "C4": {"workload": "C4: dense complex Hermitian d=4096, spectrum U[-500,0], full exp(A) (V=I), n=24",
           "d": 4096, "n": 24, "l2": "input 268 MB and 12 x 268 MB of factors exceed L2; no flush"},
    "C5": {"workload": "C5: 2-D 5-point Laplacian 512x512 (bandwidth 512), spectrum (-400,0), 8 RHS, n=16",
           "N": 262144, "kb": 512, "nrhs": 8, "n": 16, "l2": "inputs > L2; no flush"},
}


def resolve_shard(shard, workload, world):
    if shard == "auto":
        shard = {"C2": "rows", "C3": "batch"}.get(workload, "pole")
    if (shard == "rows" and workload != "C2") or (shard == "batch" and workload != "C3"):
        raise SystemExit(f"--shard {shard} does not apply to {workload}")
    return "pole" if world == 1 else shard


# ---- main ------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--cpu-calibrate", action="store_true",
                    help="time the three BASELINE.md §3 CPU thread settings for --workload and record the best")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--prof-steps", type=int, default=3)
    ap.add_argument("--shard", choices=["auto", "pole", "rows", "batch"], default="pole")
    ap.add_argument("--c1-batch", type=int, default=1,
                    help="C1 only: this many independent C1 problems per step in one call (throughput mode)")
    ap.add_argument("--no-colsplit", action="store_true",
                    help="C4 at N > 1: plain contiguous pole blocks (no column split of the leftover pairs)")
    ap.add_argument("--check", action="store_true",
                    help="after timing, compare rank 0's sharded result with an unsharded call (check_rel)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cores = os.cpu_count() or 1
    peaks = load_peaks()

    shard = resolve_shard(args.shard, args.workload, world)
    config = config_dict(args.workload, world, shard)

    if args.cpu_calibrate:
        if rank == 0:
            print(json.dumps(cpu_calibrate(args.workload, cores)), flush=True)
        return

    if args.impl == "reference":
        if rank != 0:
            return
        # the reference's own CPU implementation on all host cores (its recorded best thread
        # setting); every step is one bounded sample of the workload (oracle/cpu_timer.py),
        # median over K after W warm-up steps
        steps, warmup = max(1, args.steps), max(0, args.warmup)
        r = run_cpu(args.workload, cores, cpu_best_setting(args.workload), steps, warmup)
        value = r["value"]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
            "ms_per_step": 1e3 * r["median_step_s"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64/c128", "data": "synthetic (seeded reference recipes)",
            "impl": "reference", "config": config,
            "cpu_baseline": cpu_baseline_entry(r),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    from paper_2306_16778_b200 import _native

    # PFX_BENCH_GLOO=1 (tests only): gloo collectives on host tensors and every rank on the
    # visible GPU(s) round-robin -- exercises the multi-rank logic on a single-GPU box (the
    # ranks' kernels never wait on one another; only the host-side collectives synchronise)
    gloo = os.environ.get("PFX_BENCH_GLOO") == "1"
    local_dev = local % max(1, torch.cuda.device_count()) if gloo else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def reduce_sum(t):
        """One reduce (sum) of t to rank 0: NCCL on the device tensor (gloo: via the host)."""
        if world == 1:
            return t
        if gloo:
            h = t.cpu()
            dist.reduce(torch.view_as_real(h) if h.is_complex() else h, dst=0, op=dist.ReduceOp.SUM)
            t.copy_(h)
        else:
            # complex partials go through the collective as their (re, im) float64 view (same memory)
            dist.reduce(torch.view_as_real(t) if t.is_complex() else t, dst=0, op=dist.ReduceOp.SUM)
        return t

    def all_max(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if gloo else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    from paper_2306_16778_b200 import workloads as W

    n = {"C1": 16, "C2": 24, "C3": 20, "C4": 24, "C5": 16}[args.workload]
    npairs = n // 2
    lo, hi = (rank * npairs // world, (rank + 1) * npairs // world) if shard == "pole" else (0, npairs)
    nbatch = W.C3["batch"]
    brange = (rank * nbatch // world, (rank + 1) * nbatch // world) if shard == "batch" else None
    # C4 (dense full mode) with pairs that do not divide over the ranks: whole pairs per rank,
    # the leftover pairs split by inverse columns (sharding.colsplit_plan)
    col_tasks = None
    if args.workload == "C4" and shard == "pole" and world > 1 and npairs % world and not args.no_colsplit:
        from paper_2306_16778_b200.sharding import colsplit_plan
        col_tasks = colsplit_plan(npairs, W.C4["d"], rank, world)
        config["parallelism"] += "; leftover pairs split by inverse columns (cost-balanced)"
    if args.c1_batch > 1:
        if args.workload != "C1":
            raise SystemExit("--c1-batch applies to --workload C1")
        config["batch"] = args.c1_batch
        config["workload"] += f" x {args.c1_batch} independent problems per step (throughput mode)"
    wl = Workload(args.workload, torch, dev, lo, hi, batch_range=brange, col_tasks=col_tasks,
                  c1_batch=args.c1_batch)
    stream = torch.cuda.current_stream()

    def allgather(mine):
        """All-gather of a small float64 host block (row sharding's scan aggregates)."""
        if gloo:
            parts = [torch.empty(mine.size, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(mine))
            return torch.cat(parts).numpy()
        full = torch.empty(world * mine.size, dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(full, torch.from_numpy(mine).to(dev))
        return full.cpu().numpy()

    rows = None
    if shard == "rows":
        rows = _native.tridiag_shard_rows(1 << 20, 16, rank, world)

    def compute(st):
        """This rank's share of one eval; pole sharding adds the one reduce to rank 0."""
        if shard == "rows":
            di = wl.dev_in
            wl.out = _native.expm_tridiag_shard(di["diag"], di["off"], di["V"], wl.theta2, wl.coef2, 0.0, rank, world,
                                                allgather, out=wl.out, stream=st)
            return wl.out
        out = wl.step(st)
        return reduce_sum(out) if shard == "pole" else out

    def barrier():
        if world > 1:
            if gloo:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    def one_step(ev=None):
        # ev: (start, end) events bracketing the step's compute; the L2 flush (C1) runs
        # before the start event, i.e. between timed iterations, not inside them
        if wl.flush is not None:
            wl.flush.zero_()
        if ev is not None:
            ev[0].record(stream)
        out = compute(stream)
        if ev is not None:
            ev[1].record(stream)
        return out

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    # timed region: device events on the launching stream (library profiling off, so
    # graph-captured paths run as in production)
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    step_ev = ([(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
               if wl.flush is not None else None)
    e0.record(stream)
    for i in range(args.steps):
        one_step(step_ev[i] if step_ev else None)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    # flushing configs: the sum of the per-step event pairs (flushes excluded); otherwise the
    # whole bracket
    ms = sum(a.elapsed_time(b) for a, b in step_ev) if step_ev else e0.elapsed_time(e1)
    # kernel breakdown (dominant-kernel roofline): separate pass with per-launch CUDA events
    # on the same stream; its launch durations feed roofline.achieved
    prof_steps = max(1, min(args.steps, args.prof_steps))
    _native.prof_enable(True)
    _native.prof_read()
    for _ in range(prof_steps):
        one_step()
    torch.cuda.synchronize()
    kern = _native.prof_read()
    _native.prof_enable(False)
    ms = all_max(ms)
    ms_step = ms / args.steps
    value = wl.evals_per_step * args.steps / (ms * 1e-3)

    # end-to-end with host buffers (H2D + compute + D2H per step).  N = 1: the C-ABI host
    # entry (PFX_MEM_HOST, its own pipelined staging).  N > 1 pole sharding: every rank copies
    # the inputs in, solves its pole slice on the device, the device partials meet in one NCCL
    # reduce to rank 0, and rank 0 reads the sum back; the time is the max over ranks of the
    # wall clock between two barriers
    e2e = None
    if args.e2e_steps > 0:
        h2d, d2h = wl.h2d, wl.d2h
        if shard == "rows":
            # this rank's rows in (V, diag, the couplings at its edges), its rows of out back
            r0, r1 = rows
            o0 = max(r0 - 1, 0)
            o1 = min(r1, (1 << 20) - 1)
            pin, di = wl.pinned, wl.dev_in
            pout = wl.pinned_out.view(1 << 20, 16)
            h2d = (r1 - r0) * (16 + 1) * 8 + (o1 - o0) * 8
            d2h = (r1 - r0) * 16 * 8
            if world > 1:
                t = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64, device="cpu" if gloo else dev)
                dist.all_reduce(t)
                h2d, d2h = int(t[0].item()), int(t[1].item())

        def e2e_step():
            if shard == "rows":
                di["V"][r0:r1].copy_(pin["V"][r0:r1], non_blocking=True)
                di["diag"][r0:r1].copy_(pin["diag"][r0:r1], non_blocking=True)
                if o1 > o0:
                    di["off"][o0:o1].copy_(pin["off"][o0:o1], non_blocking=True)
                out = compute(stream)
                pout[r0:r1].copy_(out[r0:r1], non_blocking=True)
                stream.synchronize()
                return
            if world > 1 and shard == "pole":
                # one H2D of the inputs, this rank's pairs on the device, ONE reduce of the
                # device partials to rank 0, one D2H of the sum at the root
                for k, v in wl.pinned.items():
                    wl.dev_in[k].copy_(v, non_blocking=True)
                out = compute(stream)
                if rank == 0:
                    wl.pinned_out.copy_(out.reshape(-1).view(torch.float64), non_blocking=True)
                stream.synchronize()
                return
            wl.step_host()
        e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        dt = all_max(time.perf_counter() - t0)
        e2e = {"value": wl.evals_per_step * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # --check: rank 0's part of the sharded result against the same computation unsharded
    check_rel = None
    if args.check:
        out_sh = compute(stream)
        torch.cuda.synchronize()
        if rank == 0:
            full = Workload(args.workload, torch, dev, 0, npairs, c1_batch=args.c1_batch)
            ref = full.step(stream)
            torch.cuda.synchronize()
            a = out_sh.reshape(ref.shape[0], -1) if shard != "batch" else out_sh.reshape(out_sh.shape[0], -1)
            b = ref.reshape(ref.shape[0], -1)
            if shard == "rows":
                r0, r1 = rows
                a, b = a[r0:r1], b[r0:r1]
            elif shard == "batch":
                b0, b1 = brange
                b = b[b0:b1]
            check_rel = float(torch.linalg.norm(a - b) / torch.linalg.norm(b))
            del full, ref
        if world > 1:
            barrier()

    launches = sum(v[0] for v in kern.values())
    dom = DOMINANT[args.workload]
    ncu = load_ncu_summary().get(args.workload, {})
    # profile names carry a phase / variant tag ("zgemm@lu", "dense_batched_kernel@nb16x2"):
    # the dominant kernel is every launch of that kernel
    dom_cnt, dom_ms, dom_fl = 0, 0.0, 0.0
    for kname, (c_, t_, f_) in kern.items():
        if kname.split("@")[0] == dom:
            dom_cnt, dom_ms, dom_fl = dom_cnt + c_, dom_ms + t_, dom_fl + f_
    roofline = None
    if dom_cnt:
        t_launch = dom_ms / dom_cnt * 1e-3
        if dom_fl > 0:
            # the kernel declares its algorithmic flops per launch (GEMM: 8 m n k per complex product)
            flops_per_launch = dom_fl / dom_cnt
        else:
            # one launch of the dominant kernel carries the path's whole algorithmic work per step
            share = {"pole": (hi - lo) / npairs, "rows": 1.0 / world, "batch": 1.0 / world}[shard]
            if col_tasks is not None:
                share = 1.0 / world
            flops_per_launch = ALG_FLOPS[args.workload] * wl.evals_per_step * share / (dom_cnt / prof_steps)
        achieved = flops_per_launch / t_launch / 1e12
        roofline = {"bound": "tensor", "pipe": "fp64 (DMMA m8n8k4 peak, measured)", "achieved": achieved,
                    "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                    "frac": achieved / peaks["fp64_tflops"], "traffic": ncu.get("dram_bytes_per_launch"),
                    "kernel": dom,
                    "kernel_ms": dom_ms / dom_cnt, "peak_source": peaks["fp64_source"],
                    # the dominant kernel's share of all kernel time in the profiled pass (one
                    # stream there, so the launches do not overlap) and that pass's kernel time per step
                    "share_of_step": dom_ms / max(sum(v[1] for v in kern.values()), 1e-30),
                    "kernel_ms_per_step_profiled": sum(v[1] for v in kern.values()) / prof_steps,
                    "path_frac": ALG_FLOPS[args.workload] * wl.evals_per_step / (ms_step * 1e-3) / 1e12
                    / peaks["fp64_tflops"] / world,
                    "hbm_gbs_alg": ALG_BYTES[args.workload] * wl.evals_per_step / (ms_step * 1e-3) / 1e9}
        # the HBM axis the north star asks for on the structured paths: compulsory bytes of the
        # whole step and the dominant kernel's measured DRAM traffic (ncu) over its live time
        roofline["hbm_peak_gbs"] = peaks["hbm_gbs"]
        roofline["hbm_frac_alg"] = roofline["hbm_gbs_alg"] / peaks["hbm_gbs"]
        tr = ncu.get("dram_bytes_per_launch")
        roofline["dram_gbs"] = tr / t_launch / 1e9 if tr else None
        # the tensor pipe's own utilisation (ncu) beside the algorithmic fraction: the 3M complex
        # product does 6 real flops per complex multiply-add where the algorithmic count is 8
        roofline["dmma_pipe_ncu"] = ncu.get("dmma_pipe_pct", None) and ncu["dmma_pipe_pct"] / 100.0
        roofline["fp64_pipe_ncu"] = ncu.get("fp64_pipe_pct", None) and ncu["fp64_pipe_pct"] / 100.0
        roofline["ncu_source"] = ncu.get("source")
        if args.workload == "C4":
            roofline["note"] = ("the timed steps run the LU look-ahead (panel chain on a second stream beside "
                                "the trailing update); the profiled pass that times the kernels keeps one stream, "
                                "so kernel_ms are the launches' own durations")
        if args.workload == "C5":
            roofline["note"] = ("the timed steps replay the block steps as a CUDA graph on six streams; the "
                                "profiled pass that times the kernels launches them one after another on one "
                                "stream, so kernel_ms are the launches' own durations and their sum exceeds "
                                "ms_per_step; path_frac is the step-level figure")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_entry(run_cpu(args.workload, cores, cpu_best_setting(args.workload), 5, 1))
        except Exception as exc:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": cores, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64/c128", "data": "synthetic (seeded reference recipes)",
            "config": config,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches * args.steps // prof_steps,
            **({"check_rel": check_rel} if args.check else {}),
            "kernels": {k: {"launches": v[0], "total_ms": v[1], "gflop": v[2] / 1e9} for k, v in kern.items()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
