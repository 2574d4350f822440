"""Schedule sweep: H in {2,4,8} x L in {12,24,36,48} on
N GPUs, DreamDDP's scheduled partial sync vs full local SGD (FLSGD).

Run under torchrun (one rank per GPU):

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      tools/sweep.py --out gpurun_out/sweep_nN.json

Per (H, L): layer sizes from synth_profile(L, seed, balanced) (the
reference's generator, profile.cpp:188-228) scaled to --dim parameters per
worker; K = 8 workers over the N ranks; sigma = 1.  The plsgd schedule is
DFS + bubble fill on the profile measured on these GPUs (dsx_lab_profile),
FLSGD averages every layer every H-th step.  Reports iterations/s and the
exposed / total sync time per iteration of each (and of plsgd without
the bubble fill, whose extra averages are free only in the cost model).
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys
import tempfile

import numpy as np
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402
from paper_2502_11058_b200 import native as N  # noqa: E402
from paper_2502_11058_b200.lab import (Lab, LabDesc, _dsc, nccl_unique_id, profile_layers,  # noqa: E402
                                       sync_mask)


def synth_sizes(L, seed, regime, dim, rank):
    N.load_dsx()
    path = os.path.join(tempfile.mkdtemp(prefix=f"sweep_r{rank}_"), f"synth_L{L}.profile")
    if _dsc().dsc_synth_profile(path.encode(), C.c_int(L), C.c_uint64(seed), regime.encode()) != 0:
        raise RuntimeError(_dsc().dsc_last_error().decode())
    pb, _, _ = profile_layers(path)
    pb = np.asarray(pb, dtype=np.float64)
    sizes = np.maximum(2, np.round(pb / pb.sum() * dim / 2) * 2).astype(np.int64)
    return [int(x) for x in sizes]


def run_mode(lab, masks_of, H, steps, dist_):
    r = 0
    for _ in range(H):
        lab.step(bench.learning_rate(r, H), masks_of(r))
        r += 1
    lab.sync()
    lab.set_noise_horizon(steps)  # exact window: the engine generates only these steps' noise
    dist_.barrier()
    lab.record(0)
    for _ in range(steps):
        lab.step(bench.learning_rate(r, H), masks_of(r))
        r += 1
    lab.record(1)
    ms = lab.elapsed_ms(0, 1)
    lab.sync()
    lab.set_noise_horizon(-1)
    lab.set_pipeline(False)
    lab.set_instrument(True)
    per = []
    for _ in range(2 * H):
        lab.step(bench.learning_rate(r, H), masks_of(r))
        r += 1
        per.append(lab.last_step_times())
    lab.set_instrument(False)
    lab.set_pipeline(True)
    import torch
    t = torch.tensor([ms, statistics.mean(p[1] for p in per), statistics.mean(p[2] for p in per)],
                     dtype=torch.float64)
    dist_.all_reduce(t, op=dist_.ReduceOp.MAX)
    ms, sync, exposed = (float(x) for x in t)
    return {"it_per_s": round(steps / (ms * 1e-3), 2), "sync_ms_per_iter": round(sync, 5),
            "exposed_sync_ms_per_iter": round(exposed, 5),
            "exposed_sync_frac": round(exposed / sync, 4) if sync > 0 else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=4_000_000)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--regime", default="balanced")
    ap.add_argument("--H", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--L", type=int, nargs="+", default=[12, 24, 36, 48])
    ap.add_argument("--link-ratio", type=float, default=None,
                    help="throttle the sync link (dsx_lab_set_link) so the whole model's transfer "
                         "takes this multiple of the measured local step: the paper's slow-network regime")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = int(os.environ.get("LOCAL_RANK", 0))
    K = a.workers
    kl = K // world
    rows = []
    for H in a.H:
        for L in a.L:
            if L < H:
                continue
            sizes = synth_sizes(L, a.seed, a.regime, a.dim, rank)
            dim = int(sum(sizes))
            lab = Lab(LabDesc(dim=dim, block_sizes=sizes, workers_total=K, workers_local=kl,
                              worker_begin=rank * kl, sigma=a.sigma, device=dev))
            uid = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            lab.comm_init(uid[0], world, rank)
            lab.seed(a.seed)
            lab.fill(0.0)
            everything = np.ones(L + 1, dtype=np.uint8)
            lab.step(bench.learning_rate(0, H), everything)
            lab.sync()
            bw = None
            if a.link_ratio:
                t_bp, _ = lab.profile(reps=3)
                import torch
                t = torch.tensor([float(np.sum(t_bp))], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                bw = dim * 8 / (a.link_ratio * float(t[0]))
                lab.set_link(bw, 0.0)
            sets, fills, text = bench.measured_schedule(lab, sizes, H, dist, rank)
            masks = [sync_mask("partial", H, r, L, sets, fills) for r in range(H)]
            masks_nf = [sync_mask("partial", H, r, L, sets, None) for r in range(H)]
            nothing = np.zeros(L + 1, dtype=np.uint8)
            steps = max(8 * H, 24)
            plsgd = run_mode(lab, lambda r: masks[r % H], H, steps, dist)
            plsgd_nf = run_mode(lab, lambda r: masks_nf[r % H], H, steps, dist)
            # FLSGD as the paper runs it: the full average after the local step
            # (simulator.cpp:117-120), not overlapped with it
            lab.set_overlap(False)
            flsgd = run_mode(lab, lambda r: everything if (r + 1) % H == 0 else nothing, H, steps, dist)
            lab.set_overlap(True)
            lab.close()
            row = {"H": H, "L": L, "dim_per_worker": dim, "gpus": world, "workers": K,
                   "link_Bps": bw,
                   "synced_param_frac_per_step": round(float(np.mean(
                       [np.dot(m[1:], sizes) / dim for m in masks])), 4),
                   "plsgd": plsgd, "plsgd_no_fill": plsgd_nf, "flsgd": flsgd,
                   "speedup_vs_flsgd": round(plsgd["it_per_s"] / flsgd["it_per_s"], 4),
                   "speedup_no_fill_vs_flsgd": round(plsgd_nf["it_per_s"] / flsgd["it_per_s"], 4)}
            rows.append(row)
            if rank == 0:
                print(json.dumps(row), flush=True)
    if rank == 0 and a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
