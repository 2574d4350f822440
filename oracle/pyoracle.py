"""ctypes wrapper over oracle/liboracle.so (the C restatement in oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU legs of bench.py, always as the checker.  The product package
(paper_2502_11058_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")
PARITY_TOOL_REF = os.path.join(REF_DIR, "parity_tool_ref")

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _setup(_lib)
    return _lib


class MT(C.Structure):
    _fields_ = [("x", C.c_uint64 * 312), ("p", C.c_uint64)]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def _setup(L):
    L.orc_worker_rng.argtypes = [C.POINTER(MT), C.c_uint64, C.c_int]
    L.orc_mt_next.argtypes = [C.POINTER(MT)]
    L.orc_mt_next.restype = C.c_uint64
    L.orc_canonical.argtypes = [C.POINTER(MT)]
    L.orc_canonical.restype = C.c_double
    L.orc_normal_fill.argtypes = [C.POINTER(MT), C.c_double, _dp, C.c_size_t]
    L.orc_make_quadratic.argtypes = [C.c_size_t, C.c_int, C.c_double, C.c_double, _dp, _u64p]
    L.orc_learning_rate.argtypes = [C.c_longlong, C.c_double, C.c_double, C.c_int, C.c_double,
                                    C.c_int, C.c_double]
    L.orc_learning_rate.restype = C.c_double
    L.orc_sync_mask.argtypes = [C.c_int, C.c_int, C.c_longlong, C.c_int, _i32p, _i32p, _i32p,
                                _i32p, _u8p]
    L.orc_plsgd_step.argtypes = [_dp, C.POINTER(MT), C.c_int, C.c_size_t, _dp, _dp, C.c_double,
                                 _u64p, C.c_int, C.c_double, _u8p, C.POINTER(C.c_double)]
    L.orc_run_training.restype = C.c_longlong
    L.orc_run_training.argtypes = [C.c_int, C.c_int, C.c_longlong, C.c_int, C.c_int, C.c_double,
                                   C.c_double, C.c_uint64, C.c_longlong, C.c_size_t, _dp, _dp,
                                   C.c_double, _u64p, C.c_int, _i32p, _i32p, _i32p, _i32p,
                                   C.c_longlong, _i64p, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                   C.c_void_p]


MODES = {"partial": 0, "full": 1, "ssgd": 2}


def worker_rng(seed: int, worker: int) -> MT:
    mt = MT()
    lib().orc_worker_rng(C.byref(mt), seed, worker)
    return mt


def mt_state_text(mt: MT) -> str:
    """libstdc++ operator<< text of a mt19937_64 (312 words then the cursor)."""
    return " ".join(str(v) for v in list(mt.x) + [mt.p])


def normals(mt: MT, stddev: float, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().orc_normal_fill(C.byref(mt), stddev, out, n)
    return out


def make_quadratic(dim: int, blocks: int, mu: float = 1.0, beta: float = 2.0):
    curv = np.empty(dim, dtype=np.float64)
    sizes = np.empty(blocks, dtype=np.uint64)
    if lib().orc_make_quadratic(dim, blocks, mu, beta, curv, sizes) != 0:
        raise ValueError("make_quadratic: bad arguments")
    return curv, sizes


def csr(sets):
    ptr = np.zeros(len(sets) + 1, dtype=np.int32)
    idx = []
    for h, s in enumerate(sets):
        idx.extend(s)
        ptr[h + 1] = len(idx)
    return ptr, np.asarray(idx if idx else [0], dtype=np.int32)


def enp(layer_count: int, period: int):
    base, extra = divmod(layer_count, period)
    sets, nxt = [], layer_count
    for h in range(period):
        size = base + (1 if h < extra else 0)
        sets.append(list(range(nxt, nxt - size, -1)))
        nxt -= size
    return sets


def sync_mask(mode: str, period: int, r: int, layer_count: int, sets, fills=None) -> np.ndarray:
    sp, si = csr(sets)
    fp, fi = csr(fills if fills is not None else [[] for _ in sets])
    mask = np.zeros(layer_count + 1, dtype=np.uint8)
    lib().orc_sync_mask(MODES[mode], period, r, layer_count, sp, si, fp, fi, mask)
    return mask


def learning_rate(r, mu, beta, period, shift_a=0.0, constant=False, eta=0.0) -> float:
    return lib().orc_learning_rate(r, mu, beta, period, shift_a, int(constant), eta)


def plsgd_step(w: np.ndarray, rngs, curvature, optimum, sigma, block_sizes, eta, mask):
    """In-place step on w[K, dim]; returns max ||g||^2."""
    K, dim = w.shape
    arr = (MT * K)(*rngs)
    out = C.c_double(0.0)
    lib().orc_plsgd_step(w, arr, K, dim, curvature, optimum, sigma, block_sizes,
                         len(block_sizes), eta, mask, C.byref(out))
    for k in range(K):
        rngs[k] = arr[k]
    return out.value


def run_training(*, workers, period, iterations, mode="partial", constant_lr=False, eta=0.0,
                 shift_a=0.0, seed=0, log_stride=1, curvature, optimum, sigma, block_sizes,
                 sets, fills=None, return_w=False):
    dim = len(curvature)
    L = len(block_sizes)
    rows = iterations // log_stride + 2
    sp, si = csr(sets)
    fp, fi = csr(fills if fills is not None else [[] for _ in sets])
    it = np.zeros(rows, dtype=np.int64)
    gamma = np.zeros(rows)
    gpl = np.zeros(rows * L)
    lemma = np.zeros(rows)
    sub = np.zeros(rows)
    isub = np.zeros(rows)
    etas = np.zeros(rows)
    sc = np.zeros(3)
    w = np.zeros(workers * dim) if return_w else None
    n = lib().orc_run_training(workers, period, iterations, MODES[mode], int(constant_lr), eta,
                               shift_a, seed, log_stride, dim, curvature, optimum, sigma,
                               block_sizes, L, sp, si, fp, fi, rows, it, gamma, gpl, lemma, sub,
                               isub, etas, sc,
                               w.ctypes.data if w is not None else None)
    out = dict(iteration=it[:n], gamma=gamma[:n], gamma_per_layer=gpl[:n * L].reshape(n, L),
               lemma=lemma[:n], subopt=sub[:n], iterate_subopt=isub[:n], eta=etas[:n],
               g_meas=sc[0], final_subopt=sc[1], final_iterate_subopt=sc[2])
    if w is not None:
        out["w"] = w.reshape(workers, dim)
    return out
