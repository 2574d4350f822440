#!/usr/bin/env python3
"""bench.py — iterations/s of DreamDDP partial-sync local SGD on B200.

Workload (BASELINE.json configs[1], ResNet-18-shaped, 8 workers, H=5): the
reference's quadratic lab with one registered layer per layer of
tests/golden/data/resnet18_like.profile (61 blocks, param_bytes/4 coordinates
each, min 1: dim = 11,689,532 per worker), K = 8 workers, H = 5, the schedule
bubble_fill(schedule_dfs(profile, 5)) computed by this framework's
(bit-exact) scheduler, sigma = 1 (exact std::mt19937_64 + normal_distribution
noise stream reproduced on the GPU), seed 1, fp64 — the reference's own
arithmetic.  A step is one plsgd_step of all K workers (local step + scheduled
in-place averaging); value = iterations/s of the whole job.  With N GPUs
(torchrun) each rank holds K/N workers and the averaging crosses NVLink
(NCCL), so total work is fixed: "scaling": "strong".

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/parity_tool_ref: trainer.cpp compiled from /root/reference) on
the same workload, one thread (the reference is single-threaded).
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

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PROFILE = os.path.join(REPO, "tests", "golden", "data", "resnet18_like.profile")
GPT2_PROFILE = os.path.join(REPO, "tests", "golden", "data", "gpt2_small.profile")
MLP_PROFILE = os.path.join(REPO, "tests", "golden", "data", "mlp8_w1024.profile")
METRIC = "iterations/sec at 1/2/4/8 B200 vs CPU ref; exposed sync time per iteration"
REF_TOOL = os.path.join(REPO, "oracle", "_ref", "parity_tool_ref")


CONFIGS = {
    # BASELINE.json configs[1]: the headline workload
    "resnet18": {"profile": PROFILE, "workers": 8, "period": 5, "parity_steps": 10,
                 "workload": "resnet18-shaped quadratic lab (61 registered layers), 8 workers, H=5"},
    # BASELINE.json configs[2] at its parameter scale (GPT-2 small: 124,439,808
    # parameters per worker registered as embeddings + 12 blocks + ln_f)
    "gpt2": {"profile": GPT2_PROFILE, "workers": 8, "period": 4, "parity_steps": 2,
             "workload": "gpt2-small-shaped quadratic lab (14 registered layers, 124,439,808 "
                         "params/worker), 8 workers, H=4"},
    # BASELINE.json configs[0] as the real NN: 8 Linear layers (1024 wide, 10
    # classes), batch 256/worker, 4 workers, H=4, SGD momentum; bf16 tcgen05
    # GEMMs (--dtype f32: the fp32 SIMT parity path)
    "mlp": {"profile": MLP_PROFILE, "workers": 4, "period": 4, "parity_steps": 8, "nn": True,
            "widths": [1024] * 8 + [10], "batch": 256,
            "workload": "configs[0] MLP: 8 Linear layers (1024 wide -> 10 classes, 7,357,450 "
                        "params/worker), batch 256/worker, 4 workers, H=4, SGD momentum"},
    # BASELINE configs[3] at its parameter scale as an NN: a Llama-1B-shaped
    # stack (d_model 2048, ffn 5632: 48 up/down blocks + a 32000-class head,
    # 1.17 B parameters per worker, 97 registered layers), batch 4096
    # tokens/worker, partial local Adam
    "llama_mlp": {"profile": MLP_PROFILE, "workers": 4, "period": 4, "parity_steps": 0, "nn": True,
                  "widths": [2048] + [5632, 2048] * 48 + [32000], "batch": 4096, "optimizer": "adam",
                  "workload": "configs[3]-scale MLP stack: 97 Linear layers (2048 <-> 5632, 32000-class head, "
                              "1.17e9 params/worker), batch 4096/worker, 4 workers, H=4, local Adam"},
    # BASELINE configs[1] as the real network: a ResNet-18-shaped conv stack
    # (CIFAR geometry, 21 registered layers, 11.17M params/worker) on 32x32x3
    # synthetic batches, 8 workers, H=5; bf16 tcgen05 implicit-GEMM convs
    "resnet18_cnn": {"profile": PROFILE, "workers": 8, "period": 5, "parity_steps": 2, "nn": True, "cnn": True,
                     "batch": 128,
                     "workload": "configs[1] ResNet-18-shaped conv stack (CIFAR geometry, 21 registered layers, "
                                 "11,172,042 params/worker), batch 128 32x32x3/worker, 8 workers, H=5, "
                                 "SGD momentum"},
    # the same step at a compute-bound size (tensor-pipe roofline)
    "mlp_wide": {"profile": MLP_PROFILE, "workers": 4, "period": 4, "parity_steps": 0, "nn": True,
                 "widths": [4096] * 8 + [16], "batch": 2048,
                 "workload": "wide MLP: 8 Linear layers (4096 wide -> 16 classes), batch 2048/worker, "
                             "4 workers, H=4, SGD momentum"},
}


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=48)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet18", choices=sorted(CONFIGS))
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--period", type=int, default=None)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--dtype", default=None, choices=["f64", "f32", "bf16"],
                    help="lab: f64 (default) / f32; mlp: bf16 (default, tcgen05) / f32 (SIMT)")
    ap.add_argument("--optimizer", default=None, choices=["sgd", "momentum", "adam"])
    ap.add_argument("--lr", type=float, default=None)
    ap.add_argument("--profile", default=None)
    ap.add_argument("--sync-algo", default="pairwise", choices=["pairwise", "nccl_avg"])
    ap.add_argument("--no-overlap", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--parity-steps", type=int, default=None,
                    help="steps of the full-size parity pass vs the reference (default per config)")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="also skips the parity pass")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="mlp: eager launches instead of CUDA graphs")
    ap.add_argument("--schedule", default="auto", choices=["auto", "measured", "profile"],
                    help="multi-GPU: schedule from the CUDA-event profile measured on these GPUs "
                         "(auto for N>1) or from --profile's times")
    a = ap.parse_args(argv)
    c = CONFIGS[a.config]
    a.profile = a.profile or c["profile"]
    a.workers = a.workers or c["workers"]
    a.period = a.period or c["period"]
    a.parity_steps = c["parity_steps"] if a.parity_steps is None else a.parity_steps
    a.workload = c["workload"]
    a.nn = bool(c.get("nn"))
    a.cnn = bool(c.get("cnn"))
    a.widths = c.get("widths")
    a.batch = c.get("batch")
    a.dtype = a.dtype or ("bf16" if a.nn else "f64")
    if a.nn and a.dtype == "f64":
        ap.error("the MLP computes in bf16 (tensor cores) or f32")
    if not a.nn and a.dtype == "bf16":
        ap.error("the quadratic lab computes in f64 or f32")
    a.optimizer = a.optimizer or c.get("optimizer", "momentum")
    if a.lr is None:
        a.lr = {"sgd": 0.05, "momentum": 0.01, "adam": 1e-3}[a.optimizer]
    return a


# ---------------------------------------------------------------- helpers ---

class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    every 5 ms (nvidia-smi every 100 ms when NVML is unavailable)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(device))
        except Exception:
            self._nvml = None

    def sample_once(self):
        if self._nvml:
            nv, h = self._nvml
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in self.REASONS.items():
                    if bits & bit:
                        self.reasons.add(name)
                return
            except Exception:
                self._nvml = None
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.QUERY,
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            r = [x.strip() for x in out.split(",")] if out else []
            if len(r) >= 9:
                if r[1].replace(".", "").isdigit():
                    self.sm.append(float(r[1]))
                if r[2].replace(".", "").isdigit():
                    self.mx.append(float(r[2]))
                for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                    "sw_power_cap"], r[5:9]):
                    if v.lower() in ("active", "1"):
                        self.reasons.add(name)
        except Exception:
            pass

    def _loop(self):
        while not self._stop.is_set():
            self.sample_once()
            self._stop.wait(0.005 if self._nvml else 0.1)

    def start(self):
        self.sample_once()  # one sample at the start of the timed region
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.sm:
            self.sample_once()

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(args):
    from paper_2502_11058_b200.lab import lab_problem, schedule_from_profile
    sizes, dim = lab_problem(args.profile)
    sets, fills, objective, text = schedule_from_profile(args.profile, args.period, fill=True)
    return sizes, dim, sets, fills, text


def learning_rate(r: int, period: int) -> float:
    """TrainerConfig::learning_rate (trainer.cpp:126-135) for mu=1, beta=2."""
    mu, beta = 1.0, 2.0
    a = max(16.0 * (beta / mu), float(period)) + 1.0
    return 4.0 / (mu * (a + float(r)))


# ------------------------------------------------------------ reference arm ---

def reference_arm(args, world, rank):
    if rank != 0:
        return None
    steps = max(1, args.steps)
    warm = max(0, args.warmup)
    # Bound the run: the full-size reference step takes seconds (2 s at
    # sigma=1 for resnet18, ~1 min for gpt2); time one step first and cap
    # the sample at ~150 s of CPU work.
    probe = run_ref_tool(args, 1, 0)
    per_step = probe["seconds"]
    budget_s = 150.0
    steps = int(max(1, min(steps, budget_s // max(per_step, 1e-9))))
    warm = int(min(warm, 1)) if per_step < 20 else 0
    res = run_ref_tool(args, steps, warm)
    it_s = res["it_per_s"]
    line = {
        "impl": "reference",
        "metric": METRIC, "value": it_s, "unit": "iterations/s", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 / it_s, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world, res["dim"]),
        "cpu_baseline": {"value": it_s, "unit": "iterations/s", "cores": 1, "kind": "reference",
                         "sample": f"{steps} timed plsgd_step calls ({warm} warm-up) of the full "
                                   f"workload ({os.path.basename(args.profile)} blocks), reference "
                                   "trainer.cpp single thread"},
        "e2e": {"value": it_s, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    return line


def run_ref_tool(args, steps, warmup):
    """The reference's trainer.cpp (compiled from /root/reference into
    oracle/_ref) running plsgd_step on the same workload; returns its JSON
    line, including the per-worker parity digest after warmup + steps."""
    if not os.path.exists(REF_TOOL):
        raise RuntimeError("oracle/_ref/parity_tool_ref missing (built by __graft_entry__.build())")
    cmd = [REF_TOOL, "bench", "0", "0", str(args.workers), str(args.period), repr(args.sigma),
           str(args.seed), str(steps), str(warmup), "partial", "dfs", args.profile]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def workload_config(args, world, dim, schedule_src="profile"):
    sched = ("bubble_fill(schedule_dfs(profile measured on these GPUs by dsx_lab_profile, H))"
             if schedule_src == "measured" else "bubble_fill(schedule_dfs(profile, H))")
    return {"workload": args.workload, "config": args.config,
            "profile": os.path.relpath(args.profile, REPO), "workers": args.workers,
            "period": args.period, "dim_per_worker": dim, "sigma": args.sigma,
            "schedule": sched, "seed": args.seed,
            "parallelism": f"dp{world} ({args.workers // world} workers/GPU)",
            "sync_algo": args.sync_algo if world > 1 else "fused in-kernel (single GPU)",
            "l2": "working set > 126 MB L2 (no flush needed)"}


# ------------------------------------------------------------------ digest ---

def fnv1a64(text: str) -> str:
    h = 1469598103934665603
    for ch in text.encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def row_digest(w, rng_text):
    """The parity_tool's per-worker digest (tests/native/parity_tool.cpp
    cmd_bench): sequential sum and sum of squares, 64 strided samples, FNV-1a
    of the rng state's text."""
    import numpy as np
    w = np.asarray(w, dtype=np.float64)
    idx = (np.arange(64, dtype=np.int64) * (len(w) - 1)) // 63
    return {"sum": float(np.cumsum(w)[-1]), "sumsq": float(np.cumsum(w * w)[-1]),
            "rng_fnv": fnv1a64(rng_text), "samples": [float(x) for x in w[idx]]}


def compare_digests(got, want, tol):
    def rel(a, b):
        return abs(a - b) / max(abs(b), 1e-300)
    worst = {"sum": 0.0, "sumsq": 0.0, "samples": 0.0}
    rng_ok = len(got) == len(want)
    for g, w in zip(got, want):
        worst["sum"] = max(worst["sum"], rel(g["sum"], w["sum"]))
        worst["sumsq"] = max(worst["sumsq"], rel(g["sumsq"], w["sumsq"]))
        worst["samples"] = max([worst["samples"]] + [rel(a, b) for a, b in zip(g["samples"], w["samples"])])
        rng_ok = rng_ok and g["rng_fnv"] == w["rng_fnv"]
    ok = rng_ok and max(worst.values()) <= tol
    return {"ok": ok, "tolerance_rel": tol, "max_rel_row_sum": worst["sum"],
            "max_rel_row_sumsq": worst["sumsq"], "max_rel_samples": worst["samples"],
            "rng_states_exact": rng_ok}


# ------------------------------------------------------------------ our arm ---

def measured_schedule(lab, sizes, H, dist, rank, fill=True):
    import tempfile

    import numpy as np

    from paper_2502_11058_b200.lab import schedule_from_profile, write_profile
    t_bp, t_comm = lab.profile(reps=5)
    t_comm = np.where(t_comm < 0, 0.0, t_comm)
    if dist is not None:
        import torch
        t = torch.tensor(np.concatenate([t_bp, t_comm]), dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_bp, t_comm = t.numpy()[: len(sizes)], t.numpy()[len(sizes):]
    path = os.path.join(tempfile.mkdtemp(prefix=f"dreamddp_r{rank}_"), "measured.profile")
    write_profile(path, [int(s) * 8 for s in sizes], np.zeros(len(sizes)), t_bp, t_comm,
                  bandwidth=1.0, latency=0.0)
    sets, fills, _, text = schedule_from_profile(path, H, fill=fill)
    return sets, fills, text


def our_arm(args, world, rank, local_rank, dist):
    import ctypes as C

    import numpy as np

    from paper_2502_11058_b200 import native as N
    from paper_2502_11058_b200.lab import Lab, LabDesc, nccl_unique_id, sync_mask

    sizes, dim, sets, fills, _ = workload(args)
    L, H, K = len(sizes), args.period, args.workers
    if K % world:
        raise SystemExit(f"--workers {K} must be divisible by the GPU count {world}")
    kl = K // world
    lab = Lab(LabDesc(dim=dim, block_sizes=sizes, workers_total=K, workers_local=kl,
                      worker_begin=rank * kl, sigma=args.sigma, dtype=args.dtype,
                      device=local_rank))
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        algo = N.DSX_SYNC_PAIRWISE if args.sync_algo == "pairwise" else N.DSX_SYNC_NCCL_AVG
        lab.comm_init(obj[0], world, rank, algo)
    lab.set_overlap(not args.no_overlap)
    lab.seed(args.seed)
    lab.fill(0.0)
    schedule_src = args.schedule if args.schedule != "auto" else ("measured" if world > 1 else "profile")
    fixed_masks = [sync_mask("partial", H, r, L, sets, fills) for r in range(H)]
    sched_text = None
    if schedule_src == "measured":
        # DreamDDP's loop on this box: CUDA-event profile of every layer's
        # local step (with its noise read: one step runs first) and cross-rank
        # average under load, identical on all ranks (max), then the bit-exact
        # DFS + bubble-fill scheduler on it
        lab.step(learning_rate(0, H), fixed_masks[0])
        lab.sync()
        sets, fills, sched_text = measured_schedule(lab, sizes, H, dist, rank)
        lab.seed(args.seed)
        lab.fill(0.0)
    masks = [sync_mask("partial", H, r, L, sets, fills) for r in range(H)]

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_ranks(vals):
        if dist is None:
            return vals
        import torch
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t]

    def timed_window(nsteps, mask_list):
        """Exactly nsteps steps between two events on the lab stream.  The
        noise engine is drained before the window and may only generate noise
        for these nsteps steps, so the window holds exactly its own engine
        work (no batch generated before record(0), none after record(1))."""
        nonlocal r
        lab.sync()
        lab.set_noise_horizon(nsteps)
        barrier()
        lab.record(0)
        for _ in range(nsteps):
            lab.step(learning_rate(r, H), mask_list[r % H])
            r += 1
        lab.record(1)
        ms = lab.elapsed_ms(0, 1)  # waits for the last event
        lab.sync()
        lab.set_noise_horizon(-1)
        return max_ranks([ms])[0]

    r = 0
    for _ in range(max(3, args.warmup)):
        lab.step(learning_rate(r, H), masks[r % H])
        r += 1
    lab.sync()
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = lab.launches()
    ms_max = timed_window(args.steps, masks)
    clocks.stop()
    launches = lab.launches() - launches0
    barrier()
    value = args.steps / (ms_max / 1e3)

    # per-step breakdown with instrumentation (separate pass; not the timed
    # one).  Noise pipelining is switched off here so the noise engine and
    # the update kernel are each timed alone (in the timed pass they overlap).
    lab.set_pipeline(False)
    lab.set_instrument(True)
    per = []
    esz = 8 if args.dtype == "f64" else 4
    sz = np.asarray(sizes, dtype=np.float64)
    lazy = world > 1 and 1 < kl <= 8

    def update_bytes_of(m_cur, m_prev):
        """Algorithmic bytes of one step's update kernels.  Single GPU: every
        row read and written (+ noise).  Several ranks with >1 local row
        (lazy broadcast): a layer averaged last step is read once (its mean),
        a layer averaged this step writes only its subtree sum."""
        noise = kl * 8 if args.sigma > 0 else 0
        if not lazy:
            return float(dim) * (kl * 2 * esz + noise)
        cur, prev = np.asarray(m_cur[1:], bool), np.asarray(m_prev[1:], bool)
        reads = np.where(prev, 1, kl) * esz + noise
        writes = np.where(cur, 1, kl) * esz
        return float(np.dot(sz, reads + writes))

    step_bytes = []
    for _ in range(2 * H):
        step_bytes.append(update_bytes_of(masks[r % H], masks[(r - 1) % H]))
        lab.step(learning_rate(r, H), masks[r % H])
        r += 1
        per.append(lab.last_step_times())
    lab.set_instrument(False)
    lab.set_pipeline(True)
    # the engine alone: one-step runs vs the pipelined batch (jump-ahead paid
    # once per batch), per step
    eng = None
    if args.sigma > 0:
        e1, eb, nb = C.c_float(), C.c_float(), C.c_int()
        N.call("dsx_lab_engine_time", lab.h, 1, 3, C.byref(e1), C.byref(nb))
        N.call("dsx_lab_engine_time", lab.h, nb.value, 3, C.byref(eb), None)
        eng = {"run_1_step_ms": round(e1.value, 4), "batch_steps": nb.value,
               "run_batch_ms": round(eb.value, 4), "per_step_ms": round(eb.value / nb.value, 4)}

    def synced_frac(ms):
        return round(float(np.mean([np.dot(m[1:], sz) / dim for m in ms])), 4)

    schedule_info = {"source": schedule_src, "synced_param_frac_per_step": synced_frac(masks)}
    nosync = None
    if world > 1:
        # the same steps with nothing to average: what the sync adds to an
        # iteration once every overlap (update, pipelined noise engine) counts
        none = np.zeros(L + 1, dtype=np.uint8)
        nosync = timed_window(args.steps, [none] * H) / args.steps
    if schedule_src == "measured":
        schedule_info["text"] = sched_text
        # the same workload under the fixed profile's schedule, for comparison
        ms_f = timed_window(args.steps, fixed_masks)
        lab.set_pipeline(False)
        lab.set_instrument(True)
        per_f = []
        for _ in range(2 * H):
            lab.step(learning_rate(r, H), fixed_masks[r % H])
            r += 1
            per_f.append(lab.last_step_times())
        lab.set_instrument(False)
        lab.set_pipeline(True)
        sf, ef = max_ranks([statistics.mean(p[1] for p in per_f), statistics.mean(p[2] for p in per_f)])
        schedule_info["fixed_profile_schedule"] = {
            "schedule": "bubble_fill(schedule_dfs(profile, H))", "value": round(args.steps / (ms_f / 1e3), 3),
            "synced_param_frac_per_step": synced_frac(fixed_masks),
            "sync_ms_per_iter": round(sf, 5), "exposed_sync_ms_per_iter": round(ef, 5),
            "exposed_sync_frac": round(ef / sf, 4) if sf > 0 else None}
    step_ms = [p[0] for p in per]
    sync_ms = [p[1] for p in per]
    exposed_ms = [p[2] for p in per]
    noise_ms = [p[3] for p in per]
    update_ms = [p[4] for p in per]
    if dist is not None:
        sync_mean, exposed_mean = max_ranks([statistics.mean(sync_ms), statistics.mean(exposed_ms)])
    else:
        sync_mean, exposed_mean = 0.0, 0.0

    peak, peak_kind = measured_peaks()
    averaging = None
    link_peak = None
    if world > 1:
        # NVLink roofline measured now, on these GPUs: a copy with the
        # averaging kernel's access pattern (dsx_lab_link_probe)
        link_peak = lab.link_probe(5) if args.sync_algo == "pairwise" else None
    if world > 1 and sync_mean > 0:
        # cross-rank average of the synced layers: ring-convention bytes
        # 2(W-1)/W x S per rank over NVLink, S = synced bytes of the exchange row
        S = synced_frac(masks) * dim * esz
        ach = 2 * (world - 1) / world * S / (sync_mean * 1e-3) / 1e9
        lp = link_peak or None
        averaging = {"bound": "nvlink", "kernel": "p2p_average (peer-memory reduce + broadcast)",
                     "achieved": round(ach, 1), "peak": round(lp, 1) if lp else None, "unit": "GB/s",
                     "frac": round(ach / lp, 4) if lp else None,
                     "peak_kind": "measured in this run: copy kernel with the averaging access pattern "
                                  "(dsx_lab_link_probe)",
                     "synced_bytes_per_step": int(S), "sync_ms_per_iter": round(sync_mean, 5),
                     "note": "sync span includes the flag barriers and runs under the concurrent update"}

    # roofline: the dominant kernel on the path
    update_bytes = int(round(statistics.mean(step_bytes)))
    upd = statistics.mean(update_ms)
    noi = statistics.mean(noise_ms)
    # which update kernel ran (mirrors libdsx's choice): the bulk-copy kernel
    # on one GPU with engine noise, the register-staged one otherwise
    bulk = (args.sigma > 0 and args.dtype == "f64" and kl == 8
            and os.environ.get("DSX_UPD_BULK", "") != "0")
    kname = "lab_update_bulk" if bulk else "lab_update"
    dom = {"kernel": (kname + (" (fused gradient+update+average, cp.async.bulk data path)" if bulk
                               else " (fused gradient+update+average)")), "ms": upd, "bytes": update_bytes}
    achieved = dom["bytes"] / (dom["ms"] / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath) and world == 1 and args.config == "resnet18" and K == 8:
        # dram bytes per launch from the committed ncu capture of this kernel,
        # dtype and noise mode (single GPU, 8 workers, resnet18 workload)
        key = f"{kname}:{args.dtype}:sigma{1 if args.sigma > 0 else 0}"
        traffic = json.load(open(tpath)).get(key)
    # step-level roofline: the step's HBM bytes (update kernels
    # + the engine's normal writes) at the measured HBM peak; with several
    # ranks the average's NVLink bytes at the link peak measured above are
    # assumed perfectly overlapped (max).  achieved/roof = t_roof / ms_per_step.
    engine_write = float(kl * dim * 8) if args.sigma > 0 else 0.0
    t_hbm = (update_bytes + engine_write) / (peak * 1e9) * 1e3
    t_link = 0.0
    if world > 1 and link_peak:
        t_link = 2 * (world - 1) / world * synced_frac(masks) * dim * esz / (link_peak * 1e9) * 1e3
    t_roof = max(t_hbm, t_link)
    ms_step = ms_max / args.steps
    step_roof = {"t_roof_ms": round(t_roof, 5), "ms_per_step": round(ms_step, 5),
                 "frac": round(t_roof / ms_step, 4),
                 "hbm_bytes_per_step": int(update_bytes + engine_write), "t_hbm_ms": round(t_hbm, 5),
                 "t_nvlink_ms": round(t_link, 5),
                 "definition": "t_roof = max(HBM bytes of the step (update reads/writes + noise-engine "
                               "normal writes) / HBM peak, NVLink bus bytes of the average / measured "
                               "link peak); the noise engine's ALU work is not in the bound"}
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": dom["kernel"], "kernel_ms": round(dom["ms"], 4),
                "algorithmic_bytes_per_launch": dom["bytes"], "peak_kind": peak_kind,
                "step": step_roof,
                "step_breakdown_ms": {"step_serialized": round(statistics.mean(step_ms), 4),
                                      "noise_engine": round(noi, 4), "update": round(upd, 4)},
                "noise_engine": {"bound": "alu (int64 twist/temper + fp64 polar)",
                                 "ms_one_step_run": round(noi, 4), "normals_per_step": kl * dim,
                                 "batched": eng, "overlapped_with_update": True}}

    # full-size parity against the reference (its trainer.cpp compiled from
    # /root/reference): the same seed, schedule and step count from zeros;
    # per-worker digests of every worker's parameters and rng state.  Rank 0
    # runs the reference (also the CPU baseline at N=1) while the GPUs step.
    parity = None
    cpu = None
    ref_res = None
    if not args.no_cpu_baseline and args.parity_steps > 0:
        import threading as th
        ref_box = {}
        ref_thread = None
        if rank == 0:
            def _ref():
                try:
                    ref_box["res"] = run_ref_tool(args, max(1, args.parity_steps - 1),
                                                  1 if args.parity_steps > 1 else 0)
                except Exception as e:  # noqa: BLE001
                    ref_box["err"] = str(e)
            ref_thread = th.Thread(target=_ref, daemon=True)
            ref_thread.start()
        lab.seed(args.seed)
        lab.fill(0.0)
        for rr in range(args.parity_steps):
            lab.step(learning_rate(rr, H), fixed_masks[rr % H])
        lab.sync()
        mine = [row_digest(lab.get_row(k), lab.rng_text(k)) for k in range(kl)]
        if dist is not None:
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            mine = [d for part in allv for d in part]
        if rank == 0:
            ref_thread.join()
            ref_res = ref_box.get("res")
            if ref_res is None:
                parity = {"ok": None, "error": ref_box.get("err", "reference run failed")}
            else:
                tol = 1e-12 if args.dtype == "f64" else 1e-5
                parity = compare_digests(mine, ref_res["digest"], tol)
                parity.update({"steps": args.parity_steps, "workers": len(mine),
                               "schedule": "bubble_fill(schedule_dfs(profile, H))",
                               "reference": "oracle/_ref/parity_tool_ref bench (trainer.cpp compiled "
                                            "from /root/reference), same seed/schedule/steps",
                               "pipelined_engine_batches": eng["batch_steps"] if eng else None})

    # e2e through the C-ABI with HOST buffers (plsgd_step semantics: worker
    # params + rng states in and out every step)
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        import torch
        # pinned host buffers: every worker's parameters and engine state go
        # in and come back every step, one transfer each way
        host = torch.zeros((kl, dim), dtype=torch.float64, pin_memory=True)
        host_rng = torch.zeros((kl, 313), dtype=torch.int64, pin_memory=True)
        wp, rp = host.data_ptr(), host_rng.data_ptr()
        N.call("dsx_lab_get_state", lab.h, wp, rp)
        lab.sync()
        # dsx_lab_step_host: plsgd_step on host rows, transfers pipelined
        # against the update (chunk c+1 in, chunk c updated, chunk c-1 out)
        rows = (C.c_void_p * kl)(*[wp + k * dim * 8 for k in range(kl)])
        masks_c = [np.ascontiguousarray(m, dtype=np.uint8) for m in masks]
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            N.call("dsx_lab_step_host", lab.h, learning_rate(r, H), masks_c[r % H].ctypes.data, rows, rp)
            r += 1
        lab.sync()
        el = max_ranks([time.perf_counter() - t0])[0]
        rng_bytes = kl * 313 * 8
        e2e = {"value": args.e2e_steps / el, "unit": "iterations/s",
               "h2d_bytes_per_step": kl * dim * 8 + rng_bytes,
               "d2h_bytes_per_step": kl * dim * 8 + rng_bytes,
               "path": ("dsx_lab_step_host: host worker rows + rng states in/out every step, " +
                        ("chunked H2D/update/D2H overlap" if world == 1 else
                         "rows in overlapping the noise engine, multi-rank step, rows out"))}

    if rank != 0:
        lab.close()
        return None

    if world == 1 and ref_res is not None:
        n_timed = max(1, args.parity_steps - 1)
        cpu = {"value": ref_res["it_per_s"], "unit": "iterations/s", "cores": 1, "kind": "reference",
               "sample": f"{n_timed} timed plsgd_step calls (after {args.parity_steps - n_timed} warm-up) of "
                         "the full workload, reference trainer.cpp compiled from /root/reference, 1 thread "
                         "(the same run is the parity reference)"}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic",
        "config": workload_config(args, world, dim, schedule_src),
        "exposed_sync_ms_per_iter": round(exposed_mean, 5),
        "sync_ms_per_iter": round(sync_mean, 5),
        "exposed_sync_frac": round(exposed_mean / sync_mean, 4) if sync_mean > 0 else None,
        "ms_per_step_without_sync": round(nosync, 5) if nosync else None,
        "sync_added_ms_per_iter": round(ms_step - nosync, 5) if nosync else None,
        "sync_added_frac": (round((ms_step - nosync) / sync_mean, 4)
                            if nosync and sync_mean > 0 else None),
        "schedule": schedule_info, "averaging": averaging,
        "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks.summary(),
        "timing": "exactly `steps` steps between CUDA events on the lab stream; the noise engine is "
                  "drained before the window and bounded to the window's steps (dsx_lab_set_noise_horizon)",
    }
    lab.close()
    return line



# -------------------------------------------------------------- the NN arm ---

def mlp_flops_per_worker(widths, batch):
    """GEMM flops of one local step: forward, wgrad and dgrad (no dgrad into
    the input layer), 2*M*N*K each."""
    f = 0.0
    for l, (i, o) in enumerate(zip(widths[:-1], widths[1:])):
        f += 2.0 * batch * i * o * (3 if l > 0 else 2)
    return f


def mlp_data_pool(args, kl, rank, npool):
    from paper_2502_11058_b200.nn import batch_pool
    return batch_pool(args.seed, [rank * kl + k for k in range(kl)], npool, args.batch, args.widths[0],
                      args.widths[-1], int(os.environ.get("LOCAL_RANK", "0")))


def mlp_cpu_oracle(args, K, steps, masks):
    """The float64 CPU restatement (oracle/mlp_oracle.py; checker and CPU
    baseline only) on the same data: (params after `steps`, seconds of the
    timed steps after one warm-up step)."""
    from oracle.mlp_oracle import MlpOracle
    from paper_2502_11058_b200.nn import batch as make_batch
    from paper_2502_11058_b200.nn import init_params, teacher
    t = teacher(args.seed, args.widths[0], args.widths[-1])
    orc = MlpOracle(args.widths, init_params(args.seed, args.widths), K, optimizer=args.optimizer,
                    eps=1e-6 if args.optimizer == "adam" else 1e-8)
    t0 = None
    for r in range(steps):
        if r == 1:
            t0 = time.perf_counter()
        orc.step([make_batch(args.seed, k, r, args.batch, args.widths[0], t) for k in range(K)],
                 args.lr, r, masks[r % len(masks)])
    sec = time.perf_counter() - t0 if t0 is not None else None
    return orc, sec


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max(int(i.get("num_threads", 1)) for i in threadpool_info()) or 1
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def mlp_reference_arm(args, world, rank):
    """The reference has no NN: its CPU implementation of this
    path is the restatement of plsgd_step with the NN gradient
    (oracle/mlp_oracle.py, float64 numpy, all BLAS threads)."""
    if rank != 0:
        return None
    from paper_2502_11058_b200.lab import enp, sync_mask
    L, H = len(args.widths) - 1, args.period
    masks = [sync_mask("partial", H, r, L, enp(L, H)) for r in range(H)]
    steps = max(2, min(args.steps, 4)) + 1
    _, sec = mlp_cpu_oracle(args, args.workers, steps, masks)
    it_s = (steps - 1) / sec
    cores = blas_threads()
    return {"impl": "reference", "metric": METRIC, "value": it_s, "unit": "iterations/s", "n_gpus": world,
            "steps": steps - 1, "warmup": 1, "ms_per_step": 1e3 / it_s, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": mlp_config(args, world, "enp"),
            "cpu_baseline": {"value": it_s, "unit": "iterations/s", "cores": cores, "kind": "port",
                             "sample": f"{steps - 1} timed steps (1 warm-up) of all {args.workers} workers, "
                                       "oracle/mlp_oracle.py float64 numpy (the reference has no NN)"},
            "e2e": {"value": it_s, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def mlp_config(args, world, schedule_src):
    return {"workload": args.workload, "config": args.config, "widths": args.widths, "batch_per_worker": args.batch,
            "workers": args.workers, "period": args.period, "optimizer": args.optimizer, "lr": args.lr,
            "schedule": schedule_src, "seed": args.seed, "cuda_graphs": not args.no_graphs,
            "parallelism": f"dp{world} ({args.workers // world} workers/GPU)",
            "sync": ("NCCL ncclAvg in place per layer on the side stream" if world > 1 else
                     "pairwise local average kernel per layer on the side stream"),
            "l2": "activations+weights per step > L2 only for mlp_wide; mlp's working set is L2-resident "
                  "(a real training step reuses its weights)"}


def mlp_arm(args, world, rank, local_rank, dist):
    import tempfile

    import numpy as np
    import torch

    from paper_2502_11058_b200.lab import enp, nccl_unique_id, schedule_from_profile, sync_mask, write_profile
    from paper_2502_11058_b200.nn import Mlp, gemm, init_params, layer_sizes

    K, H = args.workers, args.period
    if K % world:
        raise SystemExit(f"--workers {K} must be divisible by the GPU count {world}")
    kl = K // world
    L = len(args.widths) - 1
    torch.cuda.set_device(local_rank)
    m = Mlp(args.widths, args.batch, K, workers_local=kl, worker_begin=rank * kl, dtype=args.dtype,
            optimizer=args.optimizer, eps=1e-6 if args.optimizer == "adam" else 1e-8, device=local_rank)
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        m.comm_init(obj[0], world, rank)
    init = init_params(args.seed, args.widths)
    for k in range(kl):
        m.set_params(k, init)
    # the step replays one captured CUDA graph per sync mask
    m.set_graphs(not args.no_graphs)
    npool = 8
    xs, ys = mlp_data_pool(args, kl, rank, npool)
    dx = torch.from_numpy(xs).to(f"cuda:{local_rank}")
    dy = torch.from_numpy(ys).to(f"cuda:{local_rank}")

    def use_batch(r):
        p = r % npool
        m.set_batch_ptr(dx[p].data_ptr(), dy[p].data_ptr(), True)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_ranks(vals):
        if dist is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t]

    # DreamDDP's loop: CUDA-event profile of every layer (FP, BP + update,
    # cross-worker average) -> profile v1 -> bit-exact DFS + bubble fill
    use_batch(0)
    t_fp, t_bp, t_comm = m.profile(reps=5)
    t_fp, t_bp, t_comm = (np.asarray(v) for v in (max_ranks(list(t_fp)), max_ranks(list(t_bp)),
                                                      max_ranks(list(t_comm))))
    path = os.path.join(tempfile.mkdtemp(prefix=f"dreamddp_mlp_r{rank}_"), "measured.profile")
    write_profile(path, [4 * s for s in layer_sizes(args.widths)], t_fp, t_bp, t_comm, bandwidth=1.0, latency=0.0)
    sets, fills, _, sched_text = schedule_from_profile(path, H, fill=True)
    masks = [sync_mask("partial", H, r, L, sets, fills) for r in range(H)]
    sz = np.asarray(layer_sizes(args.widths), dtype=np.float64)
    synced_frac = float(np.mean([np.dot(mk[1:], sz) / sz.sum() for mk in masks]))

    r = 0

    def run(nsteps, mask_list):
        nonlocal r
        for _ in range(nsteps):
            use_batch(r)
            m.step(args.lr, r, mask_list[r % H])
            r += 1

    def timed(nsteps, mask_list):
        m.sync()
        barrier()
        m.record(0)
        run(nsteps, mask_list)
        m.record(1)
        ms = m.elapsed_ms(0, 1)
        m.sync()
        return max_ranks([ms])[0]

    run(max(3, args.warmup), masks)
    m.sync()
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    l0 = m.launches()
    ms_max = timed(args.steps, masks)
    clocks.stop()
    launches = m.launches() - l0
    value = args.steps / (ms_max / 1e3)
    ms_step = ms_max / args.steps

    # the same steps with nothing averaged: what the sync adds
    none = np.zeros(L + 1, dtype=np.uint8)
    ms_nosync = timed(args.steps, [none] * H) / args.steps
    # per-step instrumentation: compute span, sync span, exposed sync
    m.set_instrument(True)
    per = []
    for _ in range(2 * H):
        run(1, masks)
        per.append(m.last_step_times())
    m.set_instrument(False)
    comp, span, exp_ = (max_ranks([statistics.mean(p[i] for p in per)])[0] for i in (1, 2, 3))

    # roofline: tensor pipe.  Dominant kernel = a hidden layer's forward GEMM
    # (M = batch, N = K = width, all local workers batched), timed alone with
    # CUDA events on its stream; plus the whole step's GEMM flops / step time.
    peak_tf = None
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        peak_tf, peak_kind = float(pk["bf16_tflops"]), "measured (cuBLAS bf16 burst, MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        peak_tf, peak_kind = 2250.0, "fallback nominal dense bf16"
    dev = torch.device(f"cuda:{local_rank}")
    W_ = args.widths[1]
    A = torch.randn(kl, args.batch, W_, device=dev).bfloat16()
    B = torch.randn(kl, W_, W_, device=dev).bfloat16()
    Cc = torch.empty(kl, args.batch, W_, device=dev, dtype=torch.bfloat16)
    bias = torch.zeros(kl, W_, device=dev)
    st = torch.cuda.current_stream(dev)

    def one():
        gemm(A, B, Cc, M=args.batch, N_=W_, K=W_, batch=kl, lda=W_, sA=args.batch * W_, ldb=W_, sB=W_ * W_,
             ldc=W_, sC=args.batch * W_, epi=1, relu=True, bias=bias, s_bias=W_, stream=st.cuda_stream)
    kern = None
    if args.dtype == "bf16":
        for _ in range(3):
            one()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(50):
            one()
        e1.record(st)
        torch.cuda.synchronize(dev)
        kms = e0.elapsed_time(e1) / 50
        kflops = 2.0 * args.batch * W_ * W_ * kl
        kern = {"kernel": "gemm_tc_kernel (forward, hidden layer, tcgen05 + TMA, fused bias+ReLU)",
                "shape": [args.batch, W_, W_, kl], "ms": round(kms, 5), "flops": kflops,
                "achieved": round(kflops / kms / 1e9, 1)}
    step_flops = mlp_flops_per_worker(args.widths, args.batch) * kl
    step_tf = step_flops / (ms_step * 1e-3) / 1e12
    roofline = {"bound": "tensor", "unit": "TFLOP/s", "peak": peak_tf, "peak_kind": peak_kind,
                "achieved": kern["achieved"] if kern else round(step_tf, 2),
                "frac": round((kern["achieved"] if kern else step_tf) / peak_tf, 4), "traffic": None,
                "dominant_kernel": kern,
                "step": {"gemm_flops_per_step": step_flops, "achieved": round(step_tf, 2),
                         "frac": round(step_tf / peak_tf, 4), "ms_per_step": round(ms_step, 5),
                         "t_roof_ms": round(step_flops / (peak_tf * 1e12) * 1e3, 5)}}

    # parity + CPU baseline: the float64 restatement on the same data, same
    # schedule, from the same init, 2H steps (rank 0; every rank's workers)
    parity, cpu = None, None
    if args.parity_steps > 0 and not args.no_cpu_baseline:
        pm = Mlp(args.widths, args.batch, K, workers_local=kl, worker_begin=rank * kl, dtype=args.dtype,
                 optimizer=args.optimizer, eps=1e-6 if args.optimizer == "adam" else 1e-8, device=local_rank)
        if world > 1:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            pm.comm_init(obj[0], world, rank)
        for k in range(kl):
            pm.set_params(k, init)
        for rr in range(args.parity_steps):
            p = rr % npool
            pm.set_batch_ptr(dx[p].data_ptr(), dy[p].data_ptr(), True)
            pm.step(args.lr, rr, masks[rr % H])
        pm.sync()
        mine = [pm.get_params(k) for k in range(kl)]
        pm.close()
        if dist is not None:
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            mine = [w for part in allv for w in part]
        if rank == 0:
            # the pool cycles every npool steps; the oracle regenerates step r's batch
            # as batch(seed, k, r % npool) to match
            from oracle.mlp_oracle import MlpOracle
            from paper_2502_11058_b200.nn import batch as make_batch
            from paper_2502_11058_b200.nn import teacher
            t = teacher(args.seed, args.widths[0], args.widths[-1])
            orc = MlpOracle(args.widths, init, K, optimizer=args.optimizer,
                            eps=1e-6 if args.optimizer == "adam" else 1e-8)
            t0 = time.perf_counter()
            for rr in range(args.parity_steps):
                orc.step([make_batch(args.seed, k, rr % npool, args.batch, args.widths[0], t) for k in range(K)],
                         args.lr, rr, masks[rr % H])
            sec = time.perf_counter() - t0
            errs = [float(np.linalg.norm(w - o) / np.linalg.norm(o)) for w, o in zip(mine, orc.w)]
            tol = 3e-2 if args.dtype == "bf16" else 1e-4
            parity = {"ok": max(errs) <= tol, "max_rel_l2": max(errs), "tolerance_rel_l2": tol,
                      "steps": args.parity_steps, "workers": K,
                      "reference": "oracle/mlp_oracle.py float64 restatement (parity unpinned by the reference: "
                                   "it has no NN)",
                      "note": ("bf16 tensor-core operands vs float64" if args.dtype == "bf16" else
                               "fp32 vs float64; the strict 1e-5 check runs in tests/test_gpu_nn.py")}
            cpu = {"value": args.parity_steps / sec, "unit": "iterations/s", "cores": blas_threads(),
                   "kind": "port", "sample": f"{args.parity_steps} steps of all {K} workers, oracle/mlp_oracle.py "
                                             "float64 numpy (the same run is the parity reference)"}

    # e2e: host batches (pinned) in and the loss out every step, through the
    # public step call
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        hx = torch.from_numpy(xs).pin_memory()
        hy = torch.from_numpy(ys).pin_memory()
        m.sync()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            p = r % npool
            m.set_batch_ptr(hx[p].data_ptr(), hy[p].data_ptr(), False)
            m.step(args.lr, r, masks[r % H])
            m.last_loss()
            r += 1
        m.sync()
        el = max_ranks([time.perf_counter() - t0])[0]
        e2e = {"value": args.e2e_steps / el, "unit": "iterations/s",
               "h2d_bytes_per_step": int(xs[0].nbytes + ys[0].nbytes), "d2h_bytes_per_step": 4 * kl,
               "path": "dsx_mlp_set_batch (pinned host x + labels) + dsx_mlp_step + dsx_mlp_last_loss every step"}

    if rank != 0:
        m.close()
        return None
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (N(0,1) inputs, linear-teacher labels; device-resident pool of 8 batches/worker)",
        "config": mlp_config(args, world, "measured"),
        "exposed_sync_ms_per_iter": round(exp_, 5), "sync_ms_per_iter": round(span, 5),
        "exposed_sync_frac": round(exp_ / span, 4) if span > 0 else None,
        "compute_ms_per_iter": round(comp, 5),
        "ms_per_step_without_sync": round(ms_nosync, 5),
        "sync_added_ms_per_iter": round(ms_step - ms_nosync, 5),
        "schedule": {"source": "dsx_mlp_profile -> write_profile -> schedule_dfs + bubble_fill",
                     "text": sched_text, "synced_param_frac_per_step": round(synced_frac, 4),
                     "profile_ms": {"fp": [round(x * 1e3, 4) for x in t_fp], "bp": [round(x * 1e3, 4) for x in t_bp],
                                    "comm": [round(x * 1e3, 4) for x in t_comm]}},
        "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks.summary(),
    }
    m.close()
    return line


# ------------------------------------------------------- the conv-stack arm ---

CNN_PARITY_BATCH = 4  # per worker: the float64 restatement's bounded sample


def cnn_oracle_run(args, K, steps, masks, init, bsz):
    """The float64 restatement (oracle/cnn_oracle.py; checker and CPU baseline
    only): (oracle after `steps` steps at batch bsz/worker, their seconds)."""
    from oracle.cnn_oracle import CnnOracle
    from paper_2502_11058_b200.cnn import batch as make_batch
    from paper_2502_11058_b200.cnn import teacher
    t = teacher(args.seed, 32, 3, 10)
    orc = CnnOracle(64, 32, 3, 10, init, K, optimizer=args.optimizer)
    t0 = time.perf_counter()
    for r in range(steps):
        orc.step([make_batch(args.seed, k, r, bsz, 32, 3, t) for k in range(K)], args.lr, r, masks[r % len(masks)])
    return orc, time.perf_counter() - t0


def cnn_reference_arm(args, world, rank):
    """The reference has no network: its CPU implementation of
    this path is the restatement of plsgd_step with the conv stack's gradient
    (oracle/cnn_oracle.py, float64 numpy, all BLAS threads), timed on a
    bounded sample (batch 4/worker) and scaled to the workload's batch."""
    if rank != 0:
        return None
    from paper_2502_11058_b200.lab import enp, sync_mask
    L, H = 21, args.period
    masks = [sync_mask("partial", H, r, L, enp(L, H)) for r in range(H)]
    steps = max(2, min(args.steps, 3))
    _, sec = cnn_oracle_run(args, args.workers, steps, masks, cnn_init_host(args.seed), CNN_PARITY_BATCH)
    it_s = steps / sec * CNN_PARITY_BATCH / args.batch
    cores = blas_threads()
    return {"impl": "reference", "metric": METRIC, "value": it_s, "unit": "iterations/s", "n_gpus": world,
            "steps": steps, "warmup": 0, "ms_per_step": 1e3 / it_s, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cnn_config(args, world, "enp"),
            "cpu_baseline": {"value": it_s, "unit": "iterations/s", "cores": cores, "kind": "port",
                             "sample": f"{steps} steps of all {args.workers} workers at "
                                       f"batch {CNN_PARITY_BATCH}/worker, scaled x{CNN_PARITY_BATCH}/{args.batch} "
                                       "to the workload's batch; oracle/cnn_oracle.py float64 numpy"},
            "e2e": {"value": it_s, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cnn_init_host(seed):
    """cnn_init without a device handle (the packed layout is fixed by the topology)."""
    from oracle.cnn_oracle import layer_sizes, topology
    from paper_2502_11058_b200.cnn import init_params
    convs, _, head = topology(64, 32, 8, 10)
    fan = [c["k"] * c["k"] * c["cin"] for c in convs] + [head["cin"]]
    roles = [c["role"] for c in convs] + ["head"]
    return init_params(seed, layer_sizes(64, 32, 8, 10), fan, roles)


def cnn_config(args, world, schedule_src):
    return {"workload": args.workload, "config": args.config, "batch_per_worker": args.batch,
            "workers": args.workers, "period": args.period, "optimizer": args.optimizer, "lr": args.lr,
            "schedule": schedule_src, "seed": args.seed,
            "parallelism": f"dp{world} ({args.workers // world} workers/GPU)",
            "sync": ("NCCL ncclAvg in place per layer on the side stream" if world > 1 else
                     "pairwise local average kernel per layer on the side stream"),
            "l2": "activations + im2col buffers per step (GBs) far exceed L2"}


def cnn_arm(args, world, rank, local_rank, dist):
    import tempfile

    import numpy as np
    import torch

    from paper_2502_11058_b200.cnn import Cnn, batch as make_batch, teacher
    from paper_2502_11058_b200.lab import enp, nccl_unique_id, schedule_from_profile, sync_mask, write_profile

    K, H = args.workers, args.period
    if K % world:
        raise SystemExit(f"--workers {K} must be divisible by the GPU count {world}")
    kl = K // world
    torch.cuda.set_device(local_rank)
    dev = torch.device(f"cuda:{local_rank}")

    def make(bsz):
        mm = Cnn(bsz, K, workers_local=kl, worker_begin=rank * kl, dtype=args.dtype, optimizer=args.optimizer,
                 device=local_rank)
        if world > 1:
            obj = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            mm.comm_init(obj[0], world, rank)
        return mm

    m = make(args.batch)
    L = m.L
    init = cnn_init_host(args.seed)
    for k in range(kl):
        m.set_params(k, init)
    npool = 4
    t = teacher(args.seed, 32, 3, 10)
    xs = np.empty((npool, kl, args.batch, 32, 32, 3), dtype=np.float32)
    ys = np.empty((npool, kl, args.batch), dtype=np.int32)
    for p in range(npool):
        for j in range(kl):
            xs[p, j], ys[p, j] = make_batch(args.seed, rank * kl + j, p, args.batch, 32, 3, t)
    dx = torch.from_numpy(xs).to(dev)
    dy = torch.from_numpy(ys).to(dev)

    def use_batch(r):
        p = r % npool
        m.set_batch_ptr(dx[p].data_ptr(), dy[p].data_ptr(), True)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_ranks(vals):
        if dist is None:
            return vals
        tt = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return [float(x) for x in tt]

    # DreamDDP's loop on the network: CUDA-event profile -> profile v1 -> DFS
    use_batch(0)
    t_fp, t_bp, t_comm = m.profile(reps=5)
    t_fp, t_bp, t_comm = (np.asarray(max_ranks(list(v))) for v in (t_fp, t_bp, t_comm))
    path = os.path.join(tempfile.mkdtemp(prefix=f"dreamddp_cnn_r{rank}_"), "measured.profile")
    sizes = m.layer_sizes()
    write_profile(path, [4 * s_ for s_ in sizes], t_fp, t_bp, t_comm, bandwidth=1.0, latency=0.0)
    sets, fills, _, sched_text = schedule_from_profile(path, H, fill=True)
    masks = [sync_mask("partial", H, r, L, sets, fills) for r in range(H)]
    sz = np.asarray(sizes, dtype=np.float64)
    synced_frac = float(np.mean([np.dot(mk[1:], sz) / sz.sum() for mk in masks]))

    r = 0

    def run(nsteps, mask_list):
        nonlocal r
        for _ in range(nsteps):
            use_batch(r)
            m.step(args.lr, r, mask_list[r % H])
            r += 1

    def timed(nsteps, mask_list):
        m.sync()
        barrier()
        m.record(0)
        run(nsteps, mask_list)
        m.record(1)
        ms = m.elapsed_ms(0, 1)
        m.sync()
        return max_ranks([ms])[0]

    run(max(3, args.warmup), masks)
    m.sync()
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    l0 = m.launches()
    ms_max = timed(args.steps, masks)
    clocks.stop()
    launches = m.launches() - l0
    value = args.steps / (ms_max / 1e3)
    ms_step = ms_max / args.steps
    none = np.zeros(L + 1, dtype=np.uint8)
    ms_nosync = timed(args.steps, [none] * H) / args.steps
    m.set_instrument(True)
    per = []
    for _ in range(2 * H):
        run(1, masks)
        per.append(m.last_step_times())
    m.set_instrument(False)
    comp, span, exp_ = (max_ranks([statistics.mean(p_[i] for p_ in per)])[0] for i in (1, 2, 3))

    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        peak_tf, peak_kind = float(pk["bf16_tflops"]), "measured (cuBLAS bf16 burst, MEASURED_PEAKS.json)"
    except Exception:  # noqa: BLE001
        peak_tf, peak_kind = 2250.0, "fallback nominal dense bf16"
    step_flops = m.flops_per_worker() * kl
    step_tf = step_flops / (ms_step * 1e-3) / 1e12
    roofline = {"bound": "tensor", "unit": "TFLOP/s", "peak": peak_tf, "peak_kind": peak_kind,
                "achieved": round(step_tf, 2), "frac": round(step_tf / peak_tf, 4), "traffic": None,
                "scope": "whole step: implicit-GEMM conv flops (forward, wgrad, dgrad) / step time",
                "step": {"gemm_flops_per_step": step_flops, "ms_per_step": round(ms_step, 5),
                         "t_roof_ms": round(step_flops / (peak_tf * 1e12) * 1e3, 5)}}

    # parity + CPU baseline: the float64 restatement, all K workers at batch
    # CNN_PARITY_BATCH, same schedule, same init, parity_steps steps
    parity, cpu = None, None
    if args.parity_steps > 0 and not args.no_cpu_baseline:
        pm = make(CNN_PARITY_BATCH)
        for k in range(kl):
            pm.set_params(k, init)
        for rr in range(args.parity_steps):
            bs = [make_batch(args.seed, rank * kl + j, rr, CNN_PARITY_BATCH, 32, 3, t) for j in range(kl)]
            pm.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
            pm.step(args.lr, rr, masks[rr % H])
        pm.sync()
        mine = [pm.get_params(k) for k in range(kl)]
        pm.close()
        if dist is not None:
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            mine = [w for part in allv for w in part]
        if rank == 0:
            orc, sec = cnn_oracle_run(args, K, args.parity_steps, masks, init, CNN_PARITY_BATCH)
            errs = [float(np.linalg.norm(w - o) / np.linalg.norm(o)) for w, o in zip(mine, orc.w)]
            tol = 3e-2 if args.dtype == "bf16" else 1e-4
            parity = {"ok": max(errs) <= tol, "max_rel_l2": max(errs), "tolerance_rel_l2": tol,
                      "steps": args.parity_steps, "workers": K, "batch_per_worker": CNN_PARITY_BATCH,
                      "reference": "oracle/cnn_oracle.py float64 restatement (parity unpinned by the reference: "
                                   "it has no NN)"}
            it_s = args.parity_steps / sec * CNN_PARITY_BATCH / args.batch
            cpu = {"value": it_s, "unit": "iterations/s", "cores": blas_threads(), "kind": "port",
                   "sample": f"{args.parity_steps} steps of all {K} workers at batch {CNN_PARITY_BATCH}/worker "
                             f"(oracle/cnn_oracle.py float64 numpy), scaled x{CNN_PARITY_BATCH}/{args.batch}"}

    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        hx = torch.from_numpy(xs).pin_memory()
        hy = torch.from_numpy(ys).pin_memory()
        m.sync()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            p = r % npool
            m.set_batch_ptr(hx[p].data_ptr(), hy[p].data_ptr(), False)
            m.step(args.lr, r, masks[r % H])
            m.last_loss()
            r += 1
        m.sync()
        el = max_ranks([time.perf_counter() - t0])[0]
        e2e = {"value": args.e2e_steps / el, "unit": "iterations/s",
               "h2d_bytes_per_step": int(xs[0].nbytes + ys[0].nbytes), "d2h_bytes_per_step": 4 * kl,
               "path": "dsx_cnn_set_batch (pinned host x + labels) + dsx_cnn_step + dsx_cnn_last_loss every step"}
    if rank != 0:
        m.close()
        return None
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (N(0,1) 32x32x3 images, linear-teacher labels; device-resident pool of 4 batches/worker)",
        "config": cnn_config(args, world, "measured"),
        "exposed_sync_ms_per_iter": round(exp_, 5), "sync_ms_per_iter": round(span, 5),
        "exposed_sync_frac": round(exp_ / span, 4) if span > 0 else None,
        "compute_ms_per_iter": round(comp, 5),
        "ms_per_step_without_sync": round(ms_nosync, 5),
        "sync_added_ms_per_iter": round(ms_step - ms_nosync, 5),
        "schedule": {"source": "dsx_cnn_profile -> write_profile -> schedule_dfs + bubble_fill",
                     "text": sched_text, "synced_param_frac_per_step": round(synced_frac, 4),
                     "profile_ms": {"fp": [round(x * 1e3, 4) for x in t_fp], "bp": [round(x * 1e3, 4) for x in t_bp],
                                    "comm": [round(x * 1e3, 4) for x in t_comm]}},
        "roofline": roofline, "parity": parity, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks.summary(),
    }
    m.close()
    return line


def spawn_ranks(args_argv, n):
    """`python bench.py --gpus N` without torchrun: launch N ranks on this
    node (torch.distributed.run, 127.0.0.1) and relay rank 0's line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + args_argv
    return subprocess.run(cmd).returncode


def main():
    args = parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(spawn_ranks(sys.argv[1:], args.gpus))
    world = int(env_world or "1")
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              "(torchrun --nproc-per-node N) or pass a matching --gpus", file=sys.stderr)
        sys.exit(2)
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch.distributed as dist_mod
        dist_mod.init_process_group("gloo")
        dist = dist_mod
    if args.cnn:
        line = (cnn_reference_arm(args, world, rank) if args.impl == "reference"
                else cnn_arm(args, world, rank, local_rank, dist))
    elif args.nn:
        line = (mlp_reference_arm(args, world, rank) if args.impl == "reference"
                else mlp_arm(args, world, rank, local_rank, dist))
    elif args.impl == "reference":
        line = reference_arm(args, world, rank)
    else:
        line = our_arm(args, world, rank, local_rank, dist)
    if line is not None:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
