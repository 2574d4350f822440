"""Parsers for the golden fixtures written by tests/golden/make_golden.py."""
import os
import re

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DATA = os.path.join(GOLDEN, "data")


def read(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return f.read()


def parse_steps(name):
    """Returns dict(args, rows=[(r, eta, max_g2)], w=ndarray[K,dim], rng=[text])."""
    text = read(name)
    lines = text.splitlines()
    args = lines[0][2:].split()
    rows, ws, rngs = [], {}, {}
    for ln in lines[1:]:
        if ln.startswith("r="):
            m = re.match(r"r=(\d+) eta=(\S+) max_g2=(\S+)", ln)
            rows.append((int(m.group(1)), float(m.group(2)), float(m.group(3))))
        elif ln.startswith("rng"):
            k, rest = ln[3:].split(" ", 1)
            rngs[int(k)] = rest.strip()
        elif ln.startswith("w"):
            parts = ln.split()
            ws[int(parts[0][1:])] = [float(x) for x in parts[1:]]
    K = len(ws)
    w = np.array([ws[k] for k in range(K)], dtype=np.float64)
    return dict(args=args, rows=rows, w=w, rng=[rngs[k] for k in range(K)])


def step_case(args):
    """Decodes a parity_tool `steps` argv into named fields."""
    names = ["cmd", "dim", "blocks", "workers", "period", "sigma", "seed", "iters", "mode",
             "schedule"]
    out = dict(zip(names, args))
    out["profile"] = args[10] if len(args) > 10 else ""
    for k in ("dim", "blocks", "workers", "period", "seed", "iters"):
        out[k] = int(out[k])
    out["sigma"] = float(out["sigma"])
    return out


def parse_schedule_block(text):
    """First 'dreamsched-schedule v1' block in text → (sets, fills)."""
    lines = text.splitlines()
    i = lines.index("dreamsched-schedule v1")
    H = int(re.match(r"H=(\d+)", lines[i + 1]).group(1))
    sets, fills = [], []
    for ln in lines[i + 2:i + 2 + H]:
        m = re.match(r"h=\d+: sync=\[(.*)\] fill=\[(.*)\]", ln)
        sets.append([int(x) for x in m.group(1).split(",") if x])
        fills.append([int(x) for x in m.group(2).split(",") if x])
    return sets, fills


def parse_train(name):
    text = read(name)
    summary, csv = {}, []
    for ln in text.splitlines():
        if "=" in ln and "," not in ln:
            k, v = ln.split("=", 1)
            summary[k] = float(v)
        elif ln and ln[0].isdigit():
            csv.append([float(x) for x in ln.split(",")])
    return summary, np.array(csv)


def parse_train_config(path):
    kv = {}
    for ln in open(path):
        ln = ln.split("#", 1)[0].strip()
        if ln:
            k, v = ln.split("=", 1)
            kv[k.strip()] = v.strip()
    return kv


def profile_block_sizes(path):
    """One block per profile layer, param_bytes/4 coordinates (min 1) — the
    layer registration parity_tool's lab_problem() uses."""
    sizes = []
    for ln in open(path):
        f = ln.rstrip("\n").split("\t")
        if len(f) == 6 and f[0].isdigit():
            sizes.append(max(1, int(f[2]) // 4))
    return sizes
