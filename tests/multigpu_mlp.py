"""Multi-GPU MLP script (run under torchrun, one rank per GPU): K = 4 MLP
workers split over the ranks, the scheduled layers averaged across ranks
with NCCL (ncclAvg in place, or local pairwise sum + ncclSum + 1/K with
several workers per rank) on the side stream.  Rank 0 gathers every worker's
parameters and compares them with (a) the same K workers on one GPU and
(b) the float64 restatement (oracle/mlp_oracle.py).  Prints one JSON line;
exit code 0 = pass.  Used by tests/test_gpu_multigpu_nn.py."""
import json
import os
import sys

import numpy as np
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle.mlp_oracle import MlpOracle  # noqa: E402  (checker)
from paper_2502_11058_b200.lab import enp, nccl_unique_id, sync_mask  # noqa: E402
from paper_2502_11058_b200.nn import Mlp, batch, init_params, teacher  # noqa: E402


def main():
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = int(os.environ.get("LOCAL_RANK", 0))
    widths, K, H, steps, bsz, seed, lr = [256] * 8 + [10], 4, 4, 8, 64, 3, 1e-3
    L = len(widths) - 1
    kl = K // world
    t = teacher(seed, widths[0], widths[-1])
    init = init_params(seed, widths)
    sets = enp(L, H)
    masks = [sync_mask("partial", H, r, L, sets) for r in range(steps)]
    m = Mlp(widths, bsz, K, workers_local=kl, worker_begin=rank * kl, device=dev)
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    m.comm_init(uid[0], world, rank)
    graphs = os.environ.get("DSX_TEST_GRAPHS") == "1"
    m.set_graphs(graphs)  # several ranks: compute-only graphs, NCCL averages eager behind them
    overlap = os.environ.get("DSX_TEST_OVERLAP", "1") == "1"
    m.set_overlap(overlap)  # 0: every average after the whole local step (ssgd / flsgd modes)
    for k in range(kl):
        m.set_params(k, init)
    for r in range(steps):
        bs = [batch(seed, rank * kl + k, r, bsz, widths[0], t) for k in range(kl)]
        m.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
        m.step(lr, r, masks[r])
    mine = [m.get_params(k) for k in range(kl)]
    m.close()
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    ok = True
    res = {"world": world, "workers_per_rank": kl, "graphs": graphs, "overlap": overlap}
    if rank == 0:
        got = [w for part in allp for w in part]
        one = Mlp(widths, bsz, K, device=dev)
        for k in range(K):
            one.set_params(k, init)
        orc = MlpOracle(widths, init, K)
        for r in range(steps):
            bs = [batch(seed, k, r, bsz, widths[0], t) for k in range(K)]
            one.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
            one.step(lr, r, masks[r])
            orc.step(bs, lr, r, masks[r])
        ref1 = [one.get_params(k) for k in range(K)]
        one.close()
        e_one = max(float(np.linalg.norm(g - w) / np.linalg.norm(w)) for g, w in zip(got, ref1))
        e_orc = max(float(np.linalg.norm(g - w) / np.linalg.norm(w)) for g, w in zip(got, orc.w))
        # layers averaged at the last step: identical on every worker / rank
        same = True
        for l in range(1, L + 1):
            if masks[-1][l]:
                lo, hi = orc.offsets[l - 1], orc.offsets[l]
                same = same and all(np.array_equal(g[lo:hi], got[0][lo:hi]) for g in got)
        ok = e_one <= 1e-5 and e_orc <= 1e-5 and same
        res.update({"rel_l2_vs_one_gpu": e_one, "rel_l2_vs_float64": e_orc, "synced_layers_identical": same,
                    "pass": ok})
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
