"""GPU parity: the B200 path against the reference, through the C-ABI.

* build/parity_tool (the same driver source as oracle/_ref/parity_tool_ref,
  linked against this framework's drop-in libdreamsched -> libdsx) must
  reproduce the golden outputs of the REAL reference: worker parameters after
  N plsgd_step calls, every worker's std::mt19937_64 state, per-step max
  ||g||^2, and run_training traces;
* the dsx C-ABI against the C oracle on randomized configurations (worker
  counts incl. non-powers of two, odd dims, random masks, fp64 and fp32);
* the reference's acceptance binary compiled against this library, all 10
  criteria, on the GPU.

Tolerances: fp64 parameters are compared bit-exact where the path is
bit-exact by construction (update, averaging, noise accept/reject and stream
positions); the only admitted deviation is the last ulp of log() inside the
polar transform, so parameters are checked at 1e-12 relative and the rng
states exactly.  Reductions that the reference sums sequentially (||g||^2,
divergence, objective) are parallel here: 1e-12 relative.  fp32 mode: 1e-5
relative (north_star).
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O
from tests import golden_io as G

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(REPO, "build", "parity_tool")
ACCEPT = os.path.join(REPO, "build", "acceptance")
STEP_FILES = sorted(f for f in os.listdir(G.GOLDEN) if f.startswith("steps_"))


def rel_err(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0


def run_tool(*args):
    out = subprocess.run([TOOL] + list(args), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    return out.stdout


def test_smoke():
    import __graft_entry__
    __graft_entry__.smoke()


@pytest.mark.parametrize("fname", STEP_FILES)
def test_cpp_api_steps_match_reference(fname):
    gold = G.parse_steps(fname)
    args = [a if not a.endswith(".profile") else os.path.join(G.DATA, a) for a in gold["args"]]
    lines = run_tool(*args).splitlines()
    rows, ws, rngs = [], {}, {}
    for ln in lines:
        if ln.startswith("r="):
            parts = dict(kv.split("=") for kv in ln.split())
            rows.append((int(parts["r"]), float(parts["eta"]), float(parts["max_g2"])))
        elif ln.startswith("rng"):
            k, rest = ln[3:].split(" ", 1)
            rngs[int(k)] = rest.strip()
        elif ln.startswith("w"):
            p = ln.split()
            ws[int(p[0][1:])] = [float(x) for x in p[1:]]
    assert len(rows) == len(gold["rows"])
    for (r, eta, g2), (r0, eta0, g20) in zip(rows, gold["rows"]):
        assert r == r0 and eta == eta0
        assert rel_err(g2, g20) <= 1e-12
    w = np.array([ws[k] for k in range(len(ws))])
    assert w.shape == gold["w"].shape
    assert rel_err(w, gold["w"]) <= 1e-12, fname
    for k in range(len(rngs)):
        assert rngs[k] == gold["rng"][k], f"{fname}: worker {k} stream position differs"


@pytest.mark.parametrize("cfg", ["lab_partial", "lab_full", "lab_ssgd_const"])
def test_cpp_api_run_training_matches_reference(cfg):
    text = run_tool("train", os.path.join(G.DATA, cfg + ".train"))
    gold_summary, gold_csv = G.parse_train("train_%s.txt" % cfg)
    summary, csv = {}, []
    for ln in text.splitlines():
        if "=" in ln and "," not in ln:
            k, v = ln.split("=", 1)
            summary[k] = float(v)
        elif ln and ln[0].isdigit():
            csv.append([float(x) for x in ln.split(",")])
    csv = np.array(csv)
    for k in ("final_subopt", "final_iterate_subopt", "g_meas", "gamma_mean", "gamma_max"):
        assert rel_err(summary[k], gold_summary[k]) <= 1e-10, (k, summary[k], gold_summary[k])
    assert csv.shape == gold_csv.shape
    # exact zeros (synced blocks are bit-identical across workers) stay zero
    assert np.array_equal(csv == 0.0, gold_csv == 0.0)
    nz = gold_csv != 0.0
    assert rel_err(csv[nz], gold_csv[nz]) <= 1e-9


def _random_case(rng, K, dim, L, H):
    sizes = np.full(L, dim // L, dtype=np.uint64)
    sizes[: dim % L] += 1
    sets = O.enp(L, H)
    return sizes, sets


@pytest.mark.parametrize("K,dim,L,H,sigma,dtype", [
    (1, 37, 3, 2, 1.0, "f64"), (2, 129, 4, 4, 0.5, "f64"), (3, 1001, 7, 3, 1.0, "f64"),
    (5, 4097, 9, 5, 1.0, "f64"), (8, 20000, 12, 4, 1.0, "f64"), (12, 3000, 6, 3, 2.0, "f64"),
    (8, 50000, 16, 8, 0.0, "f64"), (4, 8193, 8, 4, 1.0, "f32"), (7, 999, 5, 5, 0.0, "f32"),
])
def test_dsx_lab_against_oracle(K, dim, L, H, sigma, dtype):
    from paper_2502_11058_b200 import Lab, LabDesc
    from paper_2502_11058_b200.lab import sync_mask
    rng = np.random.default_rng(K * 1000 + dim)
    sizes, sets = _random_case(rng, K, dim, L, H)
    curv, _ = O.make_quadratic(dim, L)
    seed = int(rng.integers(1, 1 << 40))
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=sigma, dtype=dtype))
    lab.seed(seed)
    w0 = rng.normal(size=(K, dim))
    lab.set_params(w0)
    w = w0.copy()
    rngs = [O.worker_rng(seed, k) for k in range(K)]
    for r in range(3 * H):
        eta = O.learning_rate(r, 1.0, 2.0, H)
        # random extra layers on top of the schedule exercise arbitrary masks
        mask = sync_mask("partial", H, r, L, sets)
        mask[1:] |= (rng.random(L) < 0.2).astype(np.uint8)
        lab.step(eta, mask)
        g2 = O.plsgd_step(w, rngs, curv, np.ones(dim), sigma, sizes, eta, mask)
        assert rel_err(lab.max_grad_norm_sq(), g2) <= (1e-12 if dtype == "f64" else 1e-4)
    got = lab.get_params()
    tol = 1e-12 if dtype == "f64" else 1e-5
    assert rel_err(got, w) <= tol
    if sigma > 0:
        for k in range(K):
            assert lab.rng_text(k) == O.mt_state_text(rngs[k])
    lab.close()


def test_dsx_external_noise_bit_exact():
    """Update + averaging kernels alone, fed the oracle's noise: bit-exact."""
    from paper_2502_11058_b200 import Lab, LabDesc
    from paper_2502_11058_b200.lab import sync_mask
    K, dim, L, H, sigma, seed = 6, 7777, 10, 5, 1.0, 99
    curv, sizes = O.make_quadratic(dim, L)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=0.0))
    w = np.zeros((K, dim))
    rngs = [O.worker_rng(seed, k) for k in range(K)]
    sets = O.enp(L, H)
    sd = sigma / np.sqrt(dim)
    for r in range(2 * H):
        eta = O.learning_rate(r, 1.0, 2.0, H)
        mask = sync_mask("partial", H, r, L, sets)
        probe = [O.MT() for _ in range(K)]
        for k in range(K):
            C_copy = O.MT()
            C_copy.x[:] = rngs[k].x[:]
            C_copy.p = rngs[k].p
            probe[k] = C_copy
        xi = np.stack([O.normals(probe[k], sd, dim) for k in range(K)])
        lab.step_with_noise(eta, mask, xi)
        O.plsgd_step(w, rngs, curv, np.ones(dim), sigma, sizes, eta, mask)
    assert np.array_equal(lab.get_params(), w)
    lab.close()


def test_noise_engine_long_stream_exact():
    """Many generations of the device MT19937-64 + polar engine: normals and
    the final stream position equal libstdc++'s (via the oracle)."""
    from paper_2502_11058_b200 import Lab, LabDesc
    dim, seed = 100003, 5
    lab = Lab(LabDesc(dim=dim, block_sizes=[dim], workers_total=1, sigma=1.0))
    lab.seed(seed)
    lab.fill(0.0)
    g = lab.gradient(0)  # curvature*(0-1) + xi
    mt = O.worker_rng(seed, 0)
    xi = O.normals(mt, 1.0 / np.sqrt(dim), dim)
    curv, _ = O.make_quadratic(dim, 1)
    ref = curv * (0.0 - 1.0) + xi
    assert rel_err(g, ref) <= 1e-12
    assert lab.rng_text(0) == O.mt_state_text(mt)
    lab.close()


@pytest.mark.parametrize("criterion", list(range(1, 11)))
def test_reference_acceptance_on_gpu(criterion):
    if not os.path.exists(ACCEPT):
        pytest.skip("acceptance binary not built")
    out = subprocess.run([ACCEPT, "--only", str(criterion)], capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.parametrize("dim,K,advance", [(1, 1, 0), (2, 2, 1), (400001, 3, 0), (250000, 2, 3),
                                           (1234567, 1, 0)])
def test_parallel_noise_engine_segments_exact(dim, K, advance):
    """The jump-ahead engine (many segments for large dims) reproduces the
    stream exactly, including odd starting cursors (a std::mt19937_64 that
    was advanced by an odd number of draws before the step)."""
    from paper_2502_11058_b200 import Lab, LabDesc
    from paper_2502_11058_b200.lab import sync_mask
    seed = 77
    L = 4 if dim >= 4 else 1
    curv, sizes = O.make_quadratic(dim, L)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=1.0))
    rngs = [O.worker_rng(seed, k) for k in range(K)]
    for k in range(K):
        for _ in range(advance + k):
            O.lib().orc_mt_next(O.C.byref(rngs[k]))
        lab.set_rng(k, np.array(list(rngs[k].x), dtype=np.uint64), int(rngs[k].p))
    w = np.zeros((K, dim))
    lab.set_params(w)
    sets = O.enp(L, 2 if L >= 2 else 1)
    H = len(sets)
    for r in range(3):
        eta = O.learning_rate(r, 1.0, 2.0, H)
        mask = sync_mask("partial", H, r, L, sets)
        lab.step(eta, mask)
        O.plsgd_step(w, rngs, curv, np.ones(dim), 1.0, sizes, eta, mask)
    assert rel_err(lab.get_params(), w) <= 1e-12
    for k in range(K):
        assert lab.rng_text(k) == O.mt_state_text(rngs[k])
    lab.close()


@pytest.mark.parametrize("pinned,chunks", [(True, None), (False, None), (True, "1"), (True, "7")])
def test_step_host_matches_device_resident_steps(pinned, chunks, monkeypatch):
    """dsx_lab_step_host (chunked, overlapped host round trip) == set_state +
    step + get_state, bit for bit, including the rng states."""
    import ctypes as C

    import torch

    from paper_2502_11058_b200 import Lab, LabDesc
    from paper_2502_11058_b200 import native as N
    from paper_2502_11058_b200.lab import sync_mask
    if chunks:
        monkeypatch.setenv("DSX_HOST_CHUNKS", chunks)
    K, dim, L, H, seed = 8, 300007, 11, 4, 21
    curv, sizes = O.make_quadratic(dim, L)
    sets = O.enp(L, H)
    a = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=1.0))
    b = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=1.0))
    for lab in (a, b):
        lab.set_pipeline(False)
        lab.seed(seed)
    w0 = np.random.default_rng(3).normal(size=(K, dim))
    host = torch.from_numpy(w0.copy())
    if pinned:
        host = host.pin_memory()
    rng = torch.zeros((K, 313), dtype=torch.int64)
    N.call("dsx_lab_get_state", a.h, None, rng.data_ptr())
    rows = (C.c_void_p * K)(*[host.data_ptr() + k * dim * 8 for k in range(K)])
    b.set_params(w0)
    for r in range(2 * H):
        eta = O.learning_rate(r, 1.0, 2.0, H)
        mask = np.ascontiguousarray(sync_mask("partial", H, r, L, sets))
        N.call("dsx_lab_step_host", a.h, eta, mask.ctypes.data, rows, rng.data_ptr())
        b.step(eta, mask)
        assert a.max_grad_norm_sq() == b.max_grad_norm_sq()
    assert np.array_equal(host.numpy(), b.get_params())
    want = torch.zeros((K, 313), dtype=torch.int64)
    N.call("dsx_lab_get_state", b.h, None, want.data_ptr())
    assert torch.equal(rng, want)
    a.close()
    b.close()


@pytest.mark.parametrize("batch,K", [("1", 8), ("3", 8), ("8", 8), ("16", 2)])
def test_batched_engine_run_boundaries(batch, K, monkeypatch):
    """Pipelined multi-step engine runs (T steps of noise per run, the next
    run prefetched): the committed rng state after any step equals libstdc++'s,
    reading it mid-run is exact, and a host write of the state mid-run drops
    the prefetched noise (trainer.cpp:191-199 draws each step's noise where the
    previous step stopped)."""
    from paper_2502_11058_b200 import Lab, LabDesc
    from paper_2502_11058_b200.lab import sync_mask
    monkeypatch.setenv("DSX_NOISE_BATCH", batch)
    dim, L, H, seed = 30011, 5, 3, 123
    curv, sizes = O.make_quadratic(dim, L)
    sets = O.enp(L, H)
    lab = Lab(LabDesc(dim=dim, block_sizes=list(sizes), workers_total=K, sigma=1.0))
    lab.seed(seed)
    rngs = [O.worker_rng(seed, k) for k in range(K)]
    w = np.zeros((K, dim))
    lab.set_params(w)
    T = int(batch)
    steps = 2 * T + 3
    for r in range(steps):
        eta = O.learning_rate(r, 1.0, 2.0, H)
        mask = sync_mask("partial", H, r, L, sets)
        lab.step(eta, mask)
        O.plsgd_step(w, rngs, curv, np.ones(dim), 1.0, sizes, eta, mask)
        if r == T // 2 + 1:  # mid-run read of the committed state
            assert lab.rng_text(K - 1) == O.mt_state_text(rngs[K - 1])
        if r == T + 1:  # mid-run host write: advance worker 0 by 5 draws
            for _ in range(5):
                O.lib().orc_mt_next(O.C.byref(rngs[0]))
            lab.set_rng(0, np.array(list(rngs[0].x), dtype=np.uint64), int(rngs[0].p))
    assert rel_err(lab.get_params(), w) <= 1e-12
    for k in range(K):
        assert lab.rng_text(k) == O.mt_state_text(rngs[k])
    lab.close()


@pytest.mark.parametrize("K,dim", [(1, 1), (3, 999), (8, 70001)])
def test_f32_host_transfer_round_trip(K, dim):
    """fp32 labs: whole-state set/get through the HBM fp64 staging buffer and
    the narrowing/widening kernels give exactly the host double->float
    rounding (row pitch ld != dim for these sizes), per row and whole-state."""
    from paper_2502_11058_b200 import Lab, LabDesc
    rng = np.random.default_rng(dim)
    lab = Lab(LabDesc(dim=dim, block_sizes=[dim], workers_total=K, sigma=0.0, dtype="f32"))
    w = rng.normal(size=(K, dim)) * 1e3
    lab.set_params(w)
    want = w.astype(np.float32).astype(np.float64)
    assert np.array_equal(lab.get_params(), want)
    lab.step(0.0, np.zeros(2, dtype=np.uint8))
    assert np.array_equal(lab.get_params(), want)
    lab.close()
