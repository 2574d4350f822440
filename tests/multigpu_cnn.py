"""Multi-GPU conv-stack script (run under torchrun, one rank per GPU): K = 4
workers of the ResNet-18-shaped stack split over the ranks, scheduled layers
averaged across ranks with NCCL on the side stream.  Rank 0 gathers every
worker's parameters and compares them with (a) the same K workers on one GPU
and (b) the float64 restatement (oracle/cnn_oracle.py).  DSX_TEST_DTYPE=f32
(width 16, SIMT, 1e-5) or bf16 (width 64: implicit-GEMM tensor-core convs,
bf16 tolerance).  Prints one JSON line; exit code 0 = pass.  Used by
tests/test_gpu_multigpu_nn.py."""
import json
import os
import sys

import numpy as np
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle.cnn_oracle import CnnOracle, layer_sizes, topology  # noqa: E402  (checker)
from paper_2502_11058_b200.cnn import Cnn, batch, init_params, teacher  # noqa: E402
from paper_2502_11058_b200.lab import enp, nccl_unique_id, sync_mask  # noqa: E402


def main():
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = int(os.environ.get("LOCAL_RANK", 0))
    dtype = os.environ.get("DSX_TEST_DTYPE", "f32")
    width, image = (16, 16) if dtype == "f32" else (64, 16)
    K, H, steps, bsz, seed, lr = 4, 2, 4, 4, 3, (1e-3 if dtype == "f32" else 0.02)
    convs, _, head = topology(width, image, 8, 10)
    init = init_params(seed, layer_sizes(width, image, 8, 10),
                       [c["k"] * c["k"] * c["cin"] for c in convs] + [head["cin"]],
                       [c["role"] for c in convs] + ["head"])
    L = len(convs) + 1
    kl = K // world
    t = teacher(seed, image, 3, 10)
    sets = enp(L, H)
    masks = [sync_mask("partial", H, r, L, sets) for r in range(steps)]
    m = Cnn(bsz, K, workers_local=kl, worker_begin=rank * kl, width=width, image=image, dtype=dtype, device=dev)
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    m.comm_init(uid[0], world, rank)
    for k in range(kl):
        m.set_params(k, init)
    for r in range(steps):
        bs = [batch(seed, rank * kl + k, r, bsz, image, 3, t) for k in range(kl)]
        m.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
        m.step(lr, r, masks[r])
    mine = [m.get_params(k) for k in range(kl)]
    offs = m.offsets
    m.close()
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    ok = True
    res = {"world": world, "workers_per_rank": kl, "dtype": dtype}
    if rank == 0:
        got = [w for part in allp for w in part]
        one = Cnn(bsz, K, width=width, image=image, dtype=dtype, device=dev)
        for k in range(K):
            one.set_params(k, init)
        orc = CnnOracle(width, image, 3, 10, init, K)
        for r in range(steps):
            bs = [batch(seed, k, r, bsz, image, 3, t) for k in range(K)]
            one.set_batch(np.stack([b[0] for b in bs]), np.stack([b[1] for b in bs]))
            one.step(lr, r, masks[r])
            orc.step(bs, lr, r, masks[r])
        ref1 = [one.get_params(k) for k in range(K)]
        one.close()
        e_one = max(float(np.linalg.norm(g - w) / np.linalg.norm(w)) for g, w in zip(got, ref1))
        e_orc = max(float(np.linalg.norm(g - w) / np.linalg.norm(w)) for g, w in zip(got, orc.w))
        same = True
        for l in range(1, L + 1):
            if masks[-1][l]:
                lo, hi = offs[l - 1], offs[l]
                same = same and all(np.array_equal(g[lo:hi], got[0][lo:hi]) for g in got)
        tol_one, tol_orc = (1e-5, 1e-5) if dtype == "f32" else (2e-3, 2e-2)
        ok = e_one <= tol_one and e_orc <= tol_orc and same
        res.update({"rel_l2_vs_one_gpu": e_one, "rel_l2_vs_float64": e_orc, "synced_layers_identical": same,
                    "pass": ok})
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
