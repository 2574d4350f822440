"""Four-mode GPU run (ssgd / wfbp / flsgd / plsgd on the throttled link) vs the
simulator; writes gpurun_out/modes.json and the measured + simulated traces.

usage: python tools/run_modes.py [--profile tests/golden/data/resnet18_like.profile]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_11058_b200 import modes  # noqa: E402
from paper_2502_11058_b200.lab import lab_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", default="tests/golden/data/resnet18_like.profile")
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--period", type=int, default=5)
    ap.add_argument("--comm-ratio", type=float, nargs="+", default=[0.5, 1.0, 2.0, 4.0])
    ap.add_argument("--latency", type=float, default=5e-6)
    ap.add_argument("--out", default="gpurun_out/modes")
    a = ap.parse_args()
    sizes, dim = lab_problem(a.profile)
    rows = []
    for ratio in a.comm_ratio:
        out = os.path.join(a.out, f"ratio{ratio:g}")
        res = modes.run(sizes, workers=a.workers, period=a.period, latency=a.latency,
                        comm_ratio=ratio, iters=2 * a.period, out_dir=out)
        res["comm_ratio"] = ratio
        res["workload"] = os.path.basename(a.profile)
        rows.append(res)
        print(json.dumps({k: v for k, v in res.items() if k not in ("schedule", "profile")}), flush=True)
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "modes.json"), "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
