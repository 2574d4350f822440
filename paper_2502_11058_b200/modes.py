"""Four training modes on the GPU vs the simulator's prediction (SURVEY §8f
#2 and #4).

The loop the paper describes, executed for real on one B200:
  1. the CUDA-event layer profiler measures every registered layer's local
     step (dsx_lab_profile),
  2. the measured times + an alpha-beta link become a "dreamsched-profile v1"
     file (write_profile),
  3. the bit-exact scheduler turns it into the plsgd schedule
     (schedule_dfs + bubble_fill), and simulate_run predicts each mode,
  4. each mode runs on the GPU with the throttled link — ssgd (all layers
     every step, transfers after the local step), wfbp (all layers, each
     transfer as soon as its layer is done), flsgd (everything every H steps,
     after the local step), plsgd (the schedule, overlapped) — and the
     measured per-layer timeline is exported in the simulator's trace schema.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import tempfile

import numpy as np

from . import native as N
from .lab import Lab, LabDesc, _dsc, schedule_from_profile, sync_mask, write_profile

MODES = ("ssgd", "wfbp", "flsgd", "plsgd")


def simulate(profile_path: str, mode: str, period: int, iters: int):
    """simulate_run of one mode -> (makespan seconds, trace JSON text)."""
    N.load_dsx()
    lib = _dsc()
    buf = C.create_string_buffer(64 << 20)
    mk = C.c_double()
    rc = lib.dsc_simulate_trace(profile_path.encode(), mode.encode(), period, C.c_longlong(iters),
                                buf, C.c_size_t(len(buf)), C.byref(mk))
    if rc != 0:
        raise RuntimeError(lib.dsc_last_error().decode())
    return mk.value, buf.value.decode()


def compare(profile_path: str, period: int, iters: int) -> str:
    """compare_modes + write_mode_report text (the four predicted makespans,
    S1, S2)."""
    N.load_dsx()
    lib = _dsc()
    buf = C.create_string_buffer(1 << 20)
    rc = lib.dsc_compare_modes(profile_path.encode(), period, C.c_longlong(iters), buf,
                               C.c_size_t(len(buf)))
    if rc != 0:
        raise RuntimeError(lib.dsc_last_error().decode())
    return buf.value.decode()


def trace_json(mode: str, steps) -> str:
    """Measured timeline -> the simulator's trace-event JSON schema
    (simulator.cpp:186-203): complete events, microsecond ts/dur rounded half
    to even, pid = mode, tid = lane."""
    events = []
    for it, (bp, comm) in enumerate(steps, start=1):
        L = len(bp) // 2
        for l in range(L):
            events.append((bp[2 * l], bp[2 * l + 1], f"BP L{l + 1}", "compute", it, l + 1))
            if comm[2 * l] >= 0:
                events.append((comm[2 * l], comm[2 * l + 1], f"COMM L{l + 1}", "link", it, l + 1))
    events.sort(key=lambda e: e[0])
    recs = []
    for s, e, name, lane, it, layer in events:
        ts = int(round(s * 1e3))
        recs.append({"name": name, "ph": "X", "ts": ts, "dur": int(round(e * 1e3)) - ts, "pid": mode,
                     "tid": lane, "args": {"iteration": it, "layer": layer}})
    return json.dumps(recs, indent=1) + "\n"


def run(block_sizes, workers=4, period=4, bandwidth=None, latency=5e-6, comm_ratio=2.0, iters=None,
        device=0, out_dir=None, reps=5):
    """Returns {mode: {measured_s, predicted_s}} + speedups; writes traces to
    out_dir when given.  bandwidth None: chosen so the full model's transfer
    takes comm_ratio x the measured local step (a comm-bound setting, where
    the modes differ)."""
    L = len(block_sizes)
    dim = int(sum(block_sizes))
    iters = iters or 2 * period
    lab = Lab(LabDesc(dim=dim, block_sizes=list(block_sizes), workers_total=workers, sigma=0.0,
                      device=device))
    lab.seed(1)
    lab.fill(0.0)
    # profiled in the throttled mode's own shape (one launch per layer)
    lab.set_link(1e15, 0.0)
    t_bp, _ = lab.profile(reps=reps)
    if bandwidth is None:
        bandwidth = dim * 8 / max(comm_ratio * float(np.sum(t_bp)) - L * latency, 1e-6)
    tmp = tempfile.mkdtemp(prefix="dreamddp_modes_")
    prof = os.path.join(tmp, "measured.profile")
    write_profile(prof, [int(s) * 8 for s in block_sizes], np.zeros(L), t_bp, None, bandwidth,
                  latency)
    sets, fills, objective, sched_text = schedule_from_profile(prof, period)
    lab.set_link(bandwidth, latency)
    lab.set_pipeline(False)
    res = {"profile": prof, "schedule": sched_text, "layers": L, "workers": workers,
           "period": period, "bandwidth_Bps": bandwidth, "latency_s": latency, "iters": iters,
           "t_bp_total_s": float(np.sum(np.round(t_bp * 1e6) * 1e-6)), "modes": {}}
    everything = np.ones(L + 1, dtype=np.uint8)
    nothing = np.zeros(L + 1, dtype=np.uint8)
    for mode in MODES:
        predicted, sim_trace = simulate(prof, mode, period, iters)
        lab.set_overlap(mode in ("wfbp", "plsgd"))
        lab.set_instrument(True)
        steps = []
        total_ms = 0.0
        for r in range(iters):
            if mode in ("ssgd", "wfbp"):
                mask = everything
            elif mode == "flsgd":
                mask = everything if (r + 1) % period == 0 or r + 1 == iters else nothing
            else:
                mask = sync_mask("partial", period, r, L, sets, fills)
            lab.step(1e-3, mask)
            step_ms = lab.last_step_times()[0]
            total_ms += step_ms
            bp = np.empty(2 * L, dtype=np.float32)
            comm = np.empty(2 * L, dtype=np.float32)
            N.call("dsx_lab_last_timeline", lab.h, bp.ctypes.data, comm.ctypes.data)
            steps.append((bp, comm, step_ms))
        # stack the per-step timelines back to back (each step starts after
        # the previous one ended, like the simulator's iteration barrier)
        offset, stacked = 0.0, []
        for bp, comm, step_ms in steps:
            stacked.append((bp + offset, np.where(comm >= 0, comm + offset, -1.0)))
            offset += step_ms
        res["modes"][mode] = {"measured_s": total_ms * 1e-3, "predicted_s": predicted}
        if out_dir:
            os.makedirs(out_dir, exist_ok=True)
            with open(os.path.join(out_dir, f"trace_measured_{mode}.json"), "w") as f:
                f.write(trace_json(mode, stacked))
            with open(os.path.join(out_dir, f"trace_simulated_{mode}.json"), "w") as f:
                f.write(sim_trace)
    lab.set_link(0.0, 0.0)
    lab.set_instrument(False)
    lab.close()
    m = res["modes"]
    for kind in ("measured_s", "predicted_s"):
        res["S1_" + kind.split("_")[0]] = m["wfbp"][kind] / m["plsgd"][kind]
        res["S2_" + kind.split("_")[0]] = m["flsgd"][kind] / m["plsgd"][kind]
    return res


def _four_modes(m, L, sizes, dx, dy, period, lr, comm_ratio, latency, iters, reps, info):
    """The four modes on a device NN (Mlp or Cnn handle): CUDA-event profile
    -> write_profile -> schedule_dfs + bubble_fill (plsgd) and simulate_run
    (the prediction); the sync stream throttled so the whole model's transfer
    takes comm_ratio x the measured FP + BP."""
    m.set_batch_ptr(dx[0].data_ptr(), dy[0].data_ptr(), True)
    t_fp, t_bp, _ = m.profile(reps=reps)
    pbytes = [4 * s for s in sizes]
    bandwidth = float(sum(pbytes)) / max(comm_ratio * float(np.sum(t_fp) + np.sum(t_bp)) - L * latency, 1e-6)
    tmp = tempfile.mkdtemp(prefix="dreamddp_nn_modes_")
    prof = os.path.join(tmp, "measured.profile")
    write_profile(prof, pbytes, t_fp, t_bp, None, bandwidth, latency)
    sets, fills, objective, sched_text = schedule_from_profile(prof, period)
    res = dict(info)
    res.update({"profile": prof, "schedule": sched_text, "period": period, "bandwidth_Bps": bandwidth,
                "latency_s": latency, "iters": iters, "t_fp_total_s": float(np.sum(t_fp)),
                "t_bp_total_s": float(np.sum(t_bp)), "modes": {}})
    everything = np.ones(L + 1, dtype=np.uint8)
    nothing = np.zeros(L + 1, dtype=np.uint8)
    m.set_link(bandwidth, latency)
    npool = dx.shape[0]
    r_global = 0
    for mode in MODES:
        predicted, _ = simulate(prof, mode, period, iters)
        m.set_overlap(mode in ("wfbp", "plsgd"))

        def mask_of(r):
            if mode in ("ssgd", "wfbp"):
                return everything
            if mode == "flsgd":
                return everything if (r + 1) % period == 0 else nothing
            return sync_mask("partial", period, r, L, sets, fills)
        for r in range(period):  # warm-up, same mode
            m.set_batch_ptr(dx[r % npool].data_ptr(), dy[r % npool].data_ptr(), True)
            m.step(lr, r_global, mask_of(r))
            r_global += 1
        m.sync()
        m.record(0)
        for r in range(iters):
            m.set_batch_ptr(dx[r % npool].data_ptr(), dy[r % npool].data_ptr(), True)
            m.step(lr, r_global, mask_of(r))
            r_global += 1
        m.record(1)
        measured = m.elapsed_ms(0, 1) * 1e-3
        m.sync()
        res["modes"][mode] = {"measured_s": measured, "predicted_s": predicted}
    m.set_link(0.0, 0.0)
    mm = res["modes"]
    for kind in ("measured_s", "predicted_s"):
        res["S1_" + kind.split("_")[0]] = mm["wfbp"][kind] / mm["plsgd"][kind]
        res["S2_" + kind.split("_")[0]] = mm["flsgd"][kind] / mm["plsgd"][kind]
    return res


def run_mlp(widths, batch_size=256, workers=4, period=4, optimizer="adam", lr=1e-3, dtype="bf16",
            comm_ratio=2.0, latency=5e-6, iters=None, device=0, reps=5, seed=1):
    """The four modes on the NN local step (the paper's Table 1 experiment on
    a real network): a K-worker MLP on one B200 whose sync stream is a
    throttled FIFO link (dsx_mlp_set_link); the CUDA-event profile of every
    layer's FP and BP + update feeds write_profile -> schedule_dfs +
    bubble_fill (plsgd) and simulate_run (the prediction).  bandwidth is
    chosen so the whole model's transfer takes comm_ratio x the measured
    FP + BP (a communication-bound setting, like the paper's 1-20 GB/s
    Ethernet).  Returns {mode: measured_s, predicted_s} and S1 / S2."""
    import torch

    from .nn import Mlp, batch_pool, init_params, layer_sizes
    L = len(widths) - 1
    iters = iters or 4 * period
    m = Mlp(widths, batch_size, workers, dtype=dtype, optimizer=optimizer,
            eps=1e-6 if optimizer == "adam" else 1e-8, device=device)
    init = init_params(seed, widths)
    for k in range(workers):
        m.set_params(k, init)
    xs, ys = batch_pool(seed, list(range(workers)), 4, batch_size, widths[0], widths[-1], device)
    dx = torch.from_numpy(xs).to(f"cuda:{device}")
    dy = torch.from_numpy(ys).to(f"cuda:{device}")
    info = {"widths": list(widths), "batch": batch_size, "workers": workers, "optimizer": optimizer,
            "dtype": dtype}
    res = _four_modes(m, L, layer_sizes(widths), dx, dy, period, lr, comm_ratio, latency, iters, reps, info)
    m.close()
    return res


def run_cnn(batch_size=128, workers=8, period=5, optimizer="momentum", lr=0.01, comm_ratio=2.0, latency=5e-6,
            iters=None, device=0, reps=5, seed=1):
    """The four modes on the ResNet-18-shaped conv stack (BASELINE
    configs[1] as a network; the paper's main model family): K workers on one
    B200, throttled sync link, same profile -> DFS -> simulate loop as
    run_mlp."""
    import torch

    from .cnn import Cnn, batch, init_params, teacher
    iters = iters or 4 * period
    m = Cnn(batch_size, workers, dtype="bf16", optimizer=optimizer, device=device)
    roles = ["stem"]
    for s_ in range(4):
        for blk in range(2):
            roles += ["a", "b"] + (["sc"] if (s_ > 0 and blk == 0) else [])
    init = init_params(seed, m.layer_sizes(), m.fan_in, roles + ["head"])
    for k in range(workers):
        m.set_params(k, init)
    t = teacher(seed, 32, 3, 10)
    xs = np.empty((2, workers, batch_size, 32, 32, 3), dtype=np.float32)
    ys = np.empty((2, workers, batch_size), dtype=np.int32)
    for p in range(2):
        for k in range(workers):
            xs[p, k], ys[p, k] = batch(seed, k, p, batch_size, 32, 3, t)
    dx = torch.from_numpy(xs).to(f"cuda:{device}")
    dy = torch.from_numpy(ys).to(f"cuda:{device}")
    info = {"model": "resnet18-shaped conv stack (21 registered layers)", "batch": batch_size,
            "workers": workers, "optimizer": optimizer, "dtype": "bf16"}
    res = _four_modes(m, m.L, m.layer_sizes(), dx, dy, period, lr, comm_ratio, latency, iters, reps, info)
    m.close()
    return res
