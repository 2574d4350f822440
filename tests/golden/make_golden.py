"""Regenerates the golden fixtures in tests/golden/ from the REAL reference.

Runs oracle/_ref/parity_tool_ref (tests/native/parity_tool.cpp linked against
the reference library compiled by oracle/Makefile from /root/reference) and
stores its stdout.  Only runnable where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
TOOL = os.path.join(REPO, "oracle", "_ref", "parity_tool_ref")
DATA = os.path.join(HERE, "data")

# (name, argv) — argv relative to parity_tool
STEP_CASES = [
    ("steps_d12_k4_h3", ["steps", "12", "3", "4", "3", "0.5", "7", "5", "partial", "enp"]),
    ("steps_d64_k8_h4", ["steps", "64", "8", "8", "4", "1.0", "3", "20", "partial", "enp"]),
    ("steps_d65_k3_h5", ["steps", "65", "5", "3", "5", "1.0", "11", "7", "partial", "enp"]),
    ("steps_d10_k8_h5", ["steps", "10", "5", "8", "5", "1.0", "13", "5", "partial", "enp"]),
    ("steps_d33_k5_full", ["steps", "33", "4", "5", "2", "0.0", "1", "6", "full", "enp"]),
    ("steps_d16_k4_ssgd", ["steps", "16", "4", "4", "1", "1.0", "7", "10", "ssgd", "single"]),
    ("steps_d1_k2", ["steps", "1", "1", "2", "1", "1.0", "9", "4", "partial", "single"]),
    ("steps_d301_k7_h3", ["steps", "301", "6", "7", "3", "0.8", "21", "8", "partial", "enp"]),
    ("steps_d257_k1_h2", ["steps", "257", "4", "1", "2", "1.5", "2", "6", "partial", "enp"]),
    ("steps_three_layer_dfs", ["steps", "0", "0", "4", "2", "1.0", "5", "6", "partial", "dfs",
                               os.path.join(DATA, "three_layer_light.profile")]),
]
TRAIN_CASES = ["lab_partial.train", "lab_full.train", "lab_ssgd_const.train"]
PROFILE_CASES = [("resnet18_like.profile", 5), ("three_layer.profile", 2),
                 ("three_layer_light.profile", 2), ("totals_123.profile", 1),
                 ("mlp8_w1024.profile", 4)]  # BASELINE configs[0]: 8-layer MLP, H=4


def run(args):
    out = subprocess.run([TOOL] + args, check=True, capture_output=True, text=True).stdout
    # fixture paths are machine-specific; store them repo-relative
    return out.replace(DATA + "/", "")


def main():
    if not os.path.exists(TOOL):
        sys.exit("build oracle/_ref first: make -C oracle ref")
    files = {}
    for name, args in STEP_CASES:
        files[name + ".txt"] = "$ " + " ".join(a.replace(DATA + "/", "") for a in args) + "\n" + run(args)
    for cfg in TRAIN_CASES:
        files["train_" + cfg.replace(".train", ".txt")] = run(["train", os.path.join(DATA, cfg)])
    for prof, h in PROFILE_CASES:
        files["profile_%s_h%d.txt" % (prof.replace(".profile", ""), h)] = run(
            ["profile", os.path.join(DATA, prof), str(h)])
    files["trace_three_layer_plsgd.txt"] = run(["trace", os.path.join(DATA, "three_layer.profile"),
                                                "plsgd", "2", "2"])
    files["sched_fuzz_2026.txt"] = run(["sched-fuzz", "2026", "150", "40"])
    for name, text in files.items():
        with open(os.path.join(HERE, name), "w") as f:
            f.write(text)
    print("wrote", len(files), "fixtures")


if __name__ == "__main__":
    main()
