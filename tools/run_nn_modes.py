"""Four training modes (ssgd / wfbp / flsgd / plsgd) on the NN local step with
a throttled sync link, measured vs the simulator (paper Table 1 style).
Writes one JSON document to stdout."""
import json
import sys

sys.path.insert(0, ".")
from paper_2502_11058_b200 import modes  # noqa: E402

out = {}
for name, widths, bsz, ratio in [("mlp_configs0_adam", [1024] * 8 + [10], 256, 2.0),
                                 ("mlp_configs0_adam_ratio1", [1024] * 8 + [10], 256, 1.0),
                                 ("mlp_wide_adam", [4096] * 8 + [16], 2048, 2.0)] + (
        [("llama_scale_mlp_adam", [2048] + [5632, 2048] * 48 + [32000], 4096, 2.0)] if "--llama" in sys.argv else []):
    out[name] = modes.run_mlp(widths, batch_size=bsz, workers=4, period=4, optimizer="adam", lr=1e-3,
                              comm_ratio=ratio)
    r = out[name]
    print(name, {k: (round(v["measured_s"], 5), round(v["predicted_s"], 5)) for k, v in r["modes"].items()},
          "S1", round(r["S1_measured"], 3), round(r["S1_predicted"], 3), "S2", round(r["S2_measured"], 3),
          round(r["S2_predicted"], 3), file=sys.stderr, flush=True)
if "--cnn" in sys.argv:
    for name, ratio in [("resnet18_cnn_momentum", 2.0), ("resnet18_cnn_momentum_ratio1", 1.0)]:
        out[name] = r = modes.run_cnn(comm_ratio=ratio)
        print(name, {k: (round(v["measured_s"], 5), round(v["predicted_s"], 5)) for k, v in r["modes"].items()},
              "S1", round(r["S1_measured"], 3), round(r["S1_predicted"], 3), "S2", round(r["S2_measured"], 3),
              round(r["S2_predicted"], 3), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
