"""Multi-GPU parity script (run under torchrun, one rank per GPU).

K workers are split into equal contiguous ranges over the ranks; every step
averages the scheduled layers across ranks over NCCL (dsx_lab_comm_init).
Rank 0 gathers all worker parameters and rng states and compares them with
the C oracle's in-process K-worker run (trainer.cpp semantics): bit-exact
for DSX_SYNC_PAIRWISE.  Exit code 0 = pass.  Used by
tests/test_gpu_multigpu.py; also runnable by hand:

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tests/multigpu_parity.py
"""
import json
import os
import sys

import numpy as np
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import pyoracle as O  # noqa: E402
from paper_2502_11058_b200 import native as N  # noqa: E402
from paper_2502_11058_b200.lab import Lab, LabDesc, nccl_unique_id, sync_mask  # noqa: E402


def run(algo, overlap, dim=200003, L=12, K=8, H=4, sigma=1.0, seed=5, steps=7):
    world, rank = dist.get_world_size(), dist.get_rank()
    kl = K // world
    curv, sizes = O.make_quadratic(dim, L)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, workers_local=kl,
                      worker_begin=rank * kl, sigma=sigma, device=int(os.environ.get("LOCAL_RANK", 0))))
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    lab.comm_init(uid[0], world, rank, algo)
    lab.set_overlap(overlap)
    lab.seed(seed)
    lab.fill(0.0)
    sets = O.enp(L, H)
    for r in range(steps):
        lab.step(O.learning_rate(r, 1.0, 2.0, H), sync_mask("partial", H, r, L, sets))
    w = lab.get_params()
    rngs = [lab.rng_text(k) for k in range(kl)]
    lab.close()
    gathered = [None] * world
    dist.all_gather_object(gathered, (w, rngs))
    if rank != 0:
        return None
    W = np.concatenate([g[0] for g in gathered])
    R = [t for g in gathered for t in g[1]]
    # the same K workers on one GPU (in-kernel averaging, same device noise)
    one = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=sigma,
                      device=int(os.environ.get("LOCAL_RANK", 0))))
    one.seed(seed)
    one.fill(0.0)
    for r in range(steps):
        one.step(O.learning_rate(r, 1.0, 2.0, H), sync_mask("partial", H, r, L, sets))
    W1 = one.get_params()
    one.close()
    ref = np.zeros((K, dim))
    orngs = [O.worker_rng(seed, k) for k in range(K)]
    for r in range(steps):
        eta = O.learning_rate(r, 1.0, 2.0, H)
        O.plsgd_step(ref, orngs, curv, np.ones(dim), sigma, sizes, eta,
                     O.sync_mask("partial", H, r, L, sets))
    err = float(np.max(np.abs(W - ref) / np.maximum(np.abs(ref), 1e-300)))
    rng_ok = all(R[k] == O.mt_state_text(orngs[k]) for k in range(K))
    # vs the oracle: equal up to the last ulp of log() in the polar transform
    # (CUDA's vs glibc's); vs the single-GPU run (same device noise): the
    # cross-rank averaging itself must be bit-identical.
    return {"algo": algo, "overlap": overlap, "max_rel_err_vs_oracle": err,
            "bit_exact_vs_single_gpu": bool(np.array_equal(W, W1)),
            "max_rel_err_vs_single_gpu": float(np.max(np.abs(W - W1) / np.maximum(np.abs(W1), 1e-300))),
            "rng_exact": rng_ok}


def _train_log(lab, L, H, sets, iters, stride):
    """run_training's loop (trainer.cpp:286-301) over the lab API: w_hat
    accumulation before every step, Gamma^l / f(w_hat) / f(mean) rows."""
    g, fh, fm = lab.log(0.0)
    rows, weight_total = [np.concatenate([g, [fh, fm]])], 0.0
    for r in range(iters):
        p_r = (3.0 + r) * (3.0 + r)
        lab.mean_accumulate(p_r)
        weight_total += p_r
        lab.step(O.learning_rate(r, 1.0, 2.0, H), sync_mask("partial", H, r, L, sets))
        if (r + 1) % stride == 0 or r + 1 == iters:
            g, fh, fm = lab.log(weight_total)
            rows.append(np.concatenate([g, [fh, fm]]))
    return np.array(rows)


def run_train_log(K=8, dim=100003, L=10, H=3, sigma=1.0, seed=9, iters=7, stride=2):
    """Multi-rank run_training logging vs the same loop on
    one GPU: the worker mean is exact on both, the Gamma partials are summed
    in a different order (<= 1e-10 relative)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    kl = K // world
    dev = int(os.environ.get("LOCAL_RANK", 0))
    _, sizes = O.make_quadratic(dim, L)
    sets = O.enp(L, H)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, workers_local=kl,
                      worker_begin=rank * kl, sigma=sigma, device=dev))
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    lab.comm_init(uid[0], world, rank)
    lab.seed(seed)
    lab.fill(0.0)
    multi = _train_log(lab, L, H, sets, iters, stride)
    lab.close()
    if rank != 0:
        return None
    one = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=sigma, device=dev))
    one.seed(seed)
    one.fill(0.0)
    single = _train_log(one, L, H, sets, iters, stride)
    one.close()
    err = float(np.max(np.abs(multi - single) / np.maximum(np.abs(single), 1e-300)))
    return {"case": "run_training_log", "K": K, "rows": int(single.shape[0]),
            "max_rel_err_vs_single_gpu": err,
            "pass": err <= 1e-10 and bool(np.all(single[:, -2:] > 0)) and bool(np.any(single[1:, :L] > 0))}


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    results = []
    world = dist.get_world_size()
    cases = [(N.DSX_SYNC_PAIRWISE, True, 8), (N.DSX_SYNC_PAIRWISE, False, 8),
             (N.DSX_SYNC_NCCL_AVG, True, 8),
             (N.DSX_SYNC_PAIRWISE, True, world)]  # one worker per GPU (in-place exchange)
    for algo, overlap, K in cases:
        res = run(algo, overlap, K=K)
        if res is not None:
            res["K"] = K
            results.append(res)
    logs = [run_train_log(K=8), run_train_log(K=world)]
    ok = True
    if dist.get_rank() == 0:
        world = dist.get_world_size()
        for res in results:
            exact_required = res["algo"] == N.DSX_SYNC_PAIRWISE or world <= 2
            res["pass"] = (res["rng_exact"] and res["max_rel_err_vs_oracle"] <= 1e-12 and
                           (res["bit_exact_vs_single_gpu"] if exact_required
                            else res["max_rel_err_vs_single_gpu"] <= 1e-12))
            ok &= res["pass"]
        for res in logs:
            results.append(res)
            ok &= res["pass"]
        print(json.dumps({"world": world, "results": results, "pass": ok}), flush=True)
    okt = [ok]
    dist.broadcast_object_list(okt, src=0)
    dist.destroy_process_group()
    sys.exit(0 if okt[0] else 1)


if __name__ == "__main__":
    main()
