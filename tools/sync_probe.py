"""Cross-GPU average throughput probe (torchrun, one rank per GPU).

Times the lab's scheduled sync of ALL layers (overlap off: pure sync span)
for each sync algorithm, next to a plain NCCL all-reduce of the same bytes."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_11058_b200 import native as N  # noqa: E402
from paper_2502_11058_b200.lab import Lab, LabDesc, lab_problem, nccl_unique_id  # noqa: E402


def main():
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    sizes, dim = lab_problem("tests/golden/data/resnet18_like.profile")
    L = len(sizes)
    out = {"world": world}
    for K in (world, 8):
        kl = K // world
        for algo_name, algo in (("pairwise_p2p", N.DSX_SYNC_PAIRWISE), ("nccl_avg", N.DSX_SYNC_NCCL_AVG)):
            lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, workers_local=kl,
                              worker_begin=rank * kl, sigma=0.0, device=dev))
            uid = [nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            lab.comm_init(uid[0], world, rank, algo)
            lab.fill(1.0)
            mask = np.ones(L + 1, dtype=np.uint8)
            res = {}
            for overlap in (False, True):
                lab.set_overlap(overlap)
                lab.set_instrument(True)
                sync, step = [], []
                for r in range(12):
                    lab.step(0.0, mask)
                    t = lab.last_step_times()
                    if r >= 2:
                        sync.append(t[1])
                        step.append(t[0])
                lab.set_instrument(False)
                s = float(np.median(sync))
                res["overlap" if overlap else "serial"] = {
                    "sync_ms": round(s, 4), "step_ms": round(float(np.median(step)), 4),
                    "algbw_GBps": round(dim * 8 / (s * 1e-3) / 1e9, 1)}
            out[f"K{K}_{algo_name}"] = res
            lab.close()
    x = torch.ones(dim, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.distributed.all_reduce  # gloo group; use a NCCL group for the device tensor
    g = dist.new_group(backend="nccl")
    for _ in range(3):
        dist.all_reduce(x, group=g)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dist.all_reduce(x, group=g)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out["torch_nccl_allreduce"] = {"ms": round(ms, 4), "algbw_GBps": round(dim * 8 / (ms * 1e-3) / 1e9, 1),
                                   "busbw_GBps": round(dim * 8 * 2 * (world - 1) / world / (ms * 1e-3) / 1e9, 1)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
