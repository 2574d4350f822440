"""Python handle over one dsx lab (include/dsx.h) plus the schedule helpers the
bench and tests need.  Mirrors the reference's trainer vocabulary: workers,
blocks (registered layers), period H, sync mask, plsgd_step.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native as N


@dataclass
class LabDesc:
    dim: int
    block_sizes: list
    workers_total: int
    workers_local: int | None = None
    worker_begin: int = 0
    sigma: float = 0.0
    dtype: str = "f64"
    device: int = 0
    curvature: np.ndarray | None = None   # default: make_quadratic(mu=1, beta=2)
    optimum: np.ndarray | None = None     # default: ones
    mu: float = 1.0
    beta: float = 2.0
    optimum_value: float = 1.0


def make_quadratic_curvature(dim: int, mu: float, beta: float) -> np.ndarray:
    """trainer.cpp:117-120, evaluated in the same order in float64."""
    if dim == 1:
        return np.array([mu])
    i = np.arange(dim, dtype=np.float64)
    return mu + (beta - mu) * i / float(dim - 1)


class Lab:
    """K (or K/N per rank) device-resident workers of the quadratic lab."""

    def __init__(self, desc: LabDesc):
        self.desc = desc
        self.dim = int(desc.dim)
        self.kl = desc.workers_local if desc.workers_local is not None else desc.workers_total
        self.L = len(desc.block_sizes)
        sizes = np.ascontiguousarray(desc.block_sizes, dtype=np.uint64)
        curv = desc.curvature if desc.curvature is not None else make_quadratic_curvature(
            self.dim, desc.mu, desc.beta)
        opt = desc.optimum if desc.optimum is not None else np.full(self.dim, desc.optimum_value)
        self._keep = (np.ascontiguousarray(sizes), np.ascontiguousarray(curv, dtype=np.float64),
                      np.ascontiguousarray(opt, dtype=np.float64))
        c = N.LabDescC()
        c.device = desc.device
        c.dtype = N.DSX_F64 if desc.dtype == "f64" else N.DSX_F32
        c.workers_total = desc.workers_total
        c.worker_begin = desc.worker_begin
        c.workers_local = self.kl
        c.dim = self.dim
        c.layers = self.L
        c.block_sizes = self._keep[0].ctypes.data_as(C.POINTER(C.c_uint64))
        c.curvature = self._keep[1].ctypes.data_as(C.POINTER(C.c_double))
        c.optimum = self._keep[2].ctypes.data_as(C.POINTER(C.c_double))
        c.noise_sigma = desc.sigma
        h = C.c_void_p()
        N.call("dsx_lab_create", C.byref(c), C.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            N.load_dsx().dsx_lab_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state -------------------------------------------------------------
    def set_params(self, w: np.ndarray) -> None:
        w = np.ascontiguousarray(w, dtype=np.float64).reshape(self.kl, self.dim)
        N.call("dsx_lab_set_all_params", self.h, w.ctypes.data)

    def get_params(self) -> np.ndarray:
        w = np.empty((self.kl, self.dim), dtype=np.float64)
        N.call("dsx_lab_get_all_params", self.h, w.ctypes.data)
        return w

    def get_row(self, local: int) -> np.ndarray:
        w = np.empty(self.dim, dtype=np.float64)
        N.call("dsx_lab_get_params", self.h, local, w.ctypes.data)
        return w

    def fill(self, value: float) -> None:
        N.call("dsx_lab_fill_params", self.h, value)

    def seed(self, seed: int) -> None:
        N.call("dsx_lab_seed_rng", self.h, seed)

    def get_rng(self, local: int):
        x = np.empty(312, dtype=np.uint64)
        p = C.c_uint64()
        N.call("dsx_lab_get_rng", self.h, local, x.ctypes.data, C.byref(p))
        return x, int(p.value)

    def set_rng(self, local: int, x, p: int) -> None:
        x = np.ascontiguousarray(x, dtype=np.uint64)
        N.call("dsx_lab_set_rng", self.h, local, x.ctypes.data, p)

    def rng_text(self, local: int) -> str:
        x, p = self.get_rng(local)
        return " ".join(str(int(v)) for v in x) + " " + str(p)

    # -- hot path ------------------------------------------------------------
    def step(self, eta: float, mask: np.ndarray) -> None:
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        N.call("dsx_lab_step", self.h, eta, mask.ctypes.data)

    def step_with_noise(self, eta: float, mask: np.ndarray, xi: np.ndarray) -> None:
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        N.call("dsx_lab_step_with_noise", self.h, eta, mask.ctypes.data, xi.ctypes.data)

    def max_grad_norm_sq(self) -> float:
        out = C.c_double()
        N.call("dsx_lab_last_max_grad_norm_sq", self.h, C.byref(out))
        return out.value

    def gradient(self, local: int = 0) -> np.ndarray:
        g = np.empty(self.dim)
        N.call("dsx_lab_gradient", self.h, local, g.ctypes.data)
        return g

    def sync(self) -> None:
        N.call("dsx_lab_sync", self.h)

    def mean_accumulate(self, weight: float) -> None:
        N.call("dsx_lab_mean_accumulate", self.h, weight)

    def log(self, weight_total: float):
        g = np.empty(self.L)
        o = np.empty(2)
        N.call("dsx_lab_log", self.h, weight_total, g.ctypes.data, o.ctypes.data)
        return g, o[0], o[1]

    # -- multi-GPU / timing ----------------------------------------------------
    def comm_init(self, uid: bytes, nranks: int, rank: int, algo: int = N.DSX_SYNC_PAIRWISE):
        buf = C.create_string_buffer(uid, 128)
        N.call("dsx_lab_comm_init", self.h, buf, nranks, rank, algo)

    def set_pipeline(self, on: bool) -> None:
        N.call("dsx_lab_set_pipeline", self.h, int(on))

    def set_noise_horizon(self, steps: int) -> None:
        """Drain the noise engine and bound its look-ahead to `steps` steps
        (-1: unbounded), so a timing window holds exactly its own engine work."""
        N.call("dsx_lab_set_noise_horizon", self.h, int(steps))

    def link_probe(self, reps: int = 5) -> float:
        """Collective: NVLink bus GB/s of a copy with the averaging kernel's
        access pattern (0 on one rank)."""
        out = C.c_double()
        N.call("dsx_lab_link_probe", self.h, reps, C.byref(out))
        return out.value

    def set_overlap(self, on: bool) -> None:
        N.call("dsx_lab_set_overlap", self.h, int(on))

    def set_instrument(self, on: bool) -> None:
        N.call("dsx_lab_set_instrument", self.h, int(on))

    def last_step_times(self):
        out = (C.c_float * 5)()
        N.call("dsx_lab_last_step_times", self.h, out)
        return tuple(out)

    def record(self, slot: int) -> None:
        N.call("dsx_lab_event_record", self.h, slot)

    def elapsed_ms(self, a: int, b: int) -> float:
        out = C.c_float()
        N.call("dsx_lab_event_elapsed", self.h, a, b, C.byref(out))
        return out.value

    def set_link(self, bandwidth: float, latency: float = 0.0) -> None:
        """Throttled sync link (bytes/s, s); bandwidth <= 0 disables."""
        N.call("dsx_lab_set_link", self.h, bandwidth, latency)

    def profile(self, reps: int = 5):
        """CUDA-event layer profiler -> (t_bp[L], t_comm[L] or -1) in seconds."""
        t_bp = np.empty(self.L)
        t_comm = np.empty(self.L)
        N.call("dsx_lab_profile", self.h, reps, t_bp.ctypes.data, t_comm.ctypes.data)
        return t_bp, t_comm

    def launches(self) -> int:
        out = C.c_uint64()
        N.call("dsx_lab_launch_count", self.h, C.byref(out))
        return int(out.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    N.call("dsx_nccl_unique_id", buf)
    return buf.raw


def device_count() -> int:
    n = C.c_int()
    N.call("dsx_device_count", C.byref(n))
    return n.value


# ---- schedules / masks (host bookkeeping, reference trainer.cpp:202-224) ----

def enp(layer_count: int, period: int):
    """Schedule::equal_number_partition (schedule.cpp:132-148)."""
    base, extra = divmod(layer_count, period)
    sets, nxt = [], layer_count
    for h in range(period):
        size = base + (1 if h < extra else 0)
        sets.append(list(range(nxt, nxt - size, -1)))
        nxt -= size
    return sets


def sync_mask(mode: str, period: int, r: int, layer_count: int, sets, fills=None) -> np.ndarray:
    mask = np.zeros(layer_count + 1, dtype=np.uint8)
    phase = (r + 1) % period
    if mode == "ssgd" or (mode == "full" and phase == 0):
        mask[:] = 1
        return mask
    if mode != "partial":
        return mask
    h = period if phase == 0 else phase
    for l in sets[h - 1]:
        mask[l] = 1
    if fills is not None and h <= len(fills):
        for l in fills[h - 1]:
            mask[l] = 1
    return mask


def schedule_masks(mode, period, layer_count, sets, fills=None):
    """The H distinct masks, indexed by (r+1) % H."""
    return [sync_mask(mode, period, r, layer_count, sets, fills) for r in range(period)]


def _dsc():
    lib = C.CDLL(N.DREAMSCHED_PATH, mode=C.RTLD_GLOBAL)
    lib.dsc_last_error.restype = C.c_char_p
    return lib


def schedule_from_profile(profile_path: str, period: int, fill: bool = True):
    """schedule_dfs + bubble_fill through libdreamsched.so -> (sets, fills, objective, text)."""
    N.load_dsx()
    lib = _dsc()
    buf = C.create_string_buffer(1 << 20)
    obj = C.c_double()
    explored = C.c_uint64()
    rc = lib.dsc_schedule_profile(profile_path.encode(), period, int(fill), buf, len(buf),
                                  C.byref(obj), C.byref(explored))
    if rc != 0:
        raise RuntimeError(lib.dsc_last_error().decode())
    text = buf.value.decode()
    sets, fills = parse_schedule_text(text)
    return sets, fills, obj.value, text


def parse_schedule_text(text: str):
    sets, fills = [], []
    for ln in text.splitlines():
        if ln.startswith("h="):
            _, rest = ln.split(": ", 1)
            sync, fill = rest.split(" ")
            sets.append([int(x) for x in sync[6:-1].split(",") if x])
            fills.append([int(x) for x in fill[6:-1].split(",") if x])
    return sets, fills


def profile_layers(profile_path: str):
    N.load_dsx()
    lib = _dsc()
    cap = 65536
    pb = (C.c_uint64 * cap)()
    fp = (C.c_double * cap)()
    bp = (C.c_double * cap)()
    cnt = C.c_int()
    rc = lib.dsc_profile_layers(profile_path.encode(), pb, fp, bp, cap, C.byref(cnt))
    if rc != 0:
        raise RuntimeError(lib.dsc_last_error().decode())
    n = cnt.value
    return list(pb[:n]), list(fp[:n]), list(bp[:n])


def lab_problem(profile_path: str):
    """Layer registration of a profile as quadratic-lab blocks: one block per
    layer, param_bytes/4 coordinates (min 1, fp32 tensors); the curvature is
    make_quadratic's (mu=1, beta=2) over the total dimension."""
    pb, _, _ = profile_layers(profile_path)
    sizes = [max(1, b // 4) for b in pb]
    return sizes, int(sum(sizes))


def write_profile(path: str, param_bytes, t_fp, t_bp, t_comm=None, bandwidth: float = 1.0,
                  latency: float = 0.0, names=None) -> None:
    """Measured per-layer times -> "dreamsched-profile v1" file through the
    drop-in library's write_profile (profile.cpp:160-174 semantics: times
    rounded to integer microseconds)."""
    N.load_dsx()
    lib = _dsc()
    L = len(param_bytes)
    pb = (C.c_uint64 * L)(*[int(x) for x in param_bytes])
    fp = (C.c_double * L)(*[float(x) for x in t_fp])
    bp = (C.c_double * L)(*[float(x) for x in t_bp])
    cm = (C.c_double * L)(*[float(x) for x in t_comm]) if t_comm is not None else None
    nm = (C.c_char_p * L)(*[(n if isinstance(n, bytes) else str(n).encode()) for n in
                            (names or [f"layer{i + 1}" for i in range(L)])])
    rc = lib.dsc_write_profile(path.encode(), L, nm, pb, fp, bp, cm, C.c_double(bandwidth),
                               C.c_double(latency))
    if rc != 0:
        raise RuntimeError(lib.dsc_last_error().decode())
