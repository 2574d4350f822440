"""Python handle over the NN local step (include/dsx_nn.h): a K-worker MLP
trained with DreamDDP's scheduled partial synchronization, plus the GEMM test
hook.  Mirrors lab.py's vocabulary (workers, registered layers, mask, step).

Data for BASELINE configs[0] ("small MLP on synthetic data"): inputs
N(0, 1), labels from a fixed random linear teacher,
one stream per (seed, worker, step) so every worker sees its own batches and
the CPU restatement (oracle/mlp_oracle.py) can regenerate them.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native as N

OPTIMIZERS = {"sgd": N.DSX_OPT_SGD, "momentum": N.DSX_OPT_MOMENTUM, "adam": N.DSX_OPT_ADAM}

# BASELINE configs[0]: 8 registered Linear layers (tests/golden/data/mlp8_w1024.profile:
# fc1..fc7 1024x1024, fc8 1024 -> 10 classes)
MLP8_WIDTHS = [1024] * 8 + [10]


def teacher(seed: int, in_dim: int, classes: int) -> np.ndarray:
    return np.random.default_rng([seed, 0x7eac]).standard_normal((classes, in_dim)).astype(np.float32)


def batch(seed: int, worker: int, step: int, size: int, in_dim: int, t: np.ndarray):
    """Worker `worker`'s batch of step `step`: x ~ N(0,1) fp32, label = argmax of the teacher."""
    rng = np.random.default_rng([seed, worker, step])
    x = rng.standard_normal((size, in_dim), dtype=np.float32)
    y = np.argmax(x.astype(np.float64) @ t.astype(np.float64).T, axis=1).astype(np.int32)
    return x, y


def batch_pool(seed: int, workers, npool: int, size: int, in_dim: int, classes: int, device: int = 0):
    """Device-resident batches [npool][len(workers)][size][in] (fp32) and
    labels [npool][len(workers)][size] (int32) for the given global worker
    ids, batch p of worker k = batch(seed, k, p).  Heads wider than 1024
    classes take the teacher's argmax on the GPU in fp32 (the float64 host
    argmax would take minutes; those configs have no CPU parity run)."""
    import torch
    dev = torch.device(f"cuda:{device}")
    t = teacher(seed, in_dim, classes)
    xs = np.empty((npool, len(workers), size, in_dim), dtype=np.float32)
    ys = np.empty((npool, len(workers), size), dtype=np.int32)
    tt = torch.from_numpy(t).to(dev) if classes > 1024 else None
    for p in range(npool):
        for j, k in enumerate(workers):
            if tt is None:
                xs[p, j], ys[p, j] = batch(seed, k, p, size, in_dim, t)
            else:
                rng = np.random.default_rng([seed, k, p])
                xs[p, j] = rng.standard_normal((size, in_dim), dtype=np.float32)
                ys[p, j] = torch.argmax(torch.from_numpy(xs[p, j]).to(dev) @ tt.T, dim=1).int().cpu().numpy()
    return xs, ys


def init_params(seed: int, widths) -> np.ndarray:
    """Packed per-worker parameters (layer l: W[out][in] then b[out]): He
    initialisation W ~ N(0, 2/in) (keeps the 8-layer ReLU stack's signal
    alive), b = 0; every worker starts from the same point (data-parallel
    initialisation)."""
    rng = np.random.default_rng([seed, 0x1a17])
    parts = []
    for i, o in zip(widths[:-1], widths[1:]):
        parts.append((rng.standard_normal(o * i) * np.sqrt(2.0 / i)).astype(np.float32))
        parts.append(np.zeros(o, dtype=np.float32))
    return np.concatenate(parts)


def layer_sizes(widths):
    """Registered-layer parameter counts (layer 1 = input side)."""
    return [i * o + o for i, o in zip(widths[:-1], widths[1:])]


class Mlp:
    """K (or K/N per rank) device-resident MLP workers."""

    def __init__(self, widths, batch_size: int, workers_total: int, workers_local: int | None = None,
                 worker_begin: int = 0, dtype: str = "f32", optimizer: str = "momentum",
                 momentum: float = 0.9, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 weight_decay: float = 0.0, device: int = 0):
        self.widths = [int(w) for w in widths]
        self.L = len(self.widths) - 1
        self.batch = int(batch_size)
        self.K = workers_total
        self.kl = workers_local if workers_local is not None else workers_total
        self.dtype = dtype
        self._w = (C.c_int * len(self.widths))(*self.widths)
        d = N.MlpDescC()
        d.device = device
        d.dtype = N.DSX_BF16 if dtype == "bf16" else N.DSX_F32
        d.workers_total = workers_total
        d.worker_begin = worker_begin
        d.workers_local = self.kl
        d.layers = self.L
        d.widths = self._w
        d.batch = self.batch
        d.optimizer = OPTIMIZERS[optimizer]
        d.momentum = momentum
        d.beta1 = beta1
        d.beta2 = beta2
        d.eps = eps
        d.weight_decay = weight_decay
        h = C.c_void_p()
        N.call("dsx_mlp_create", C.byref(d), C.byref(h))
        self.h = h
        total = C.c_uint64()
        offs = (C.c_uint64 * (self.L + 1))()
        N.call("dsx_mlp_param_layout", self.h, C.byref(total), offs)
        self.P = int(total.value)
        self.offsets = [int(x) for x in offs]
        self._keep = None

    def close(self):
        if getattr(self, "h", None):
            N.load_dsx().dsx_mlp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state ---------------------------------------------------------------
    def set_params(self, local: int, flat: np.ndarray) -> None:
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        assert flat.size == self.P
        N.call("dsx_mlp_set_params", self.h, local, flat.ctypes.data)

    def get_params(self, local: int) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        N.call("dsx_mlp_get_params", self.h, local, out.ctypes.data)
        return out

    def get_state(self, local: int):
        m = np.zeros(self.P, dtype=np.float32)
        v = np.zeros(self.P, dtype=np.float32)
        N.call("dsx_mlp_get_state", self.h, local, m.ctypes.data, v.ctypes.data)
        return m, v

    def set_batch(self, x: np.ndarray, labels: np.ndarray) -> None:
        """Host batch [kl][batch][in] fp32 + labels [kl][batch] (copied on the compute stream)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.ascontiguousarray(labels, dtype=np.int32)
        self._keep = (x, y)  # the async copy reads them
        N.call("dsx_mlp_set_batch", self.h, x.ctypes.data, y.ctypes.data, 0)

    def set_batch_ptr(self, x_ptr: int, labels_ptr: int, on_device: bool) -> None:
        N.call("dsx_mlp_set_batch", self.h, C.c_void_p(x_ptr), C.c_void_p(labels_ptr), int(on_device))

    # -- hot path --------------------------------------------------------------
    def step(self, lr: float, t: int, mask) -> None:
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        N.call("dsx_mlp_step", self.h, lr, t, mask.ctypes.data)

    def last_loss(self) -> np.ndarray:
        out = np.empty(self.kl, dtype=np.float32)
        N.call("dsx_mlp_last_loss", self.h, out.ctypes.data)
        return out

    def sync(self) -> None:
        N.call("dsx_mlp_sync", self.h)

    # -- multi-GPU / timing ------------------------------------------------------
    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        buf = C.create_string_buffer(uid, 128)
        N.call("dsx_mlp_comm_init", self.h, buf, nranks, rank)

    def set_instrument(self, on: bool) -> None:
        N.call("dsx_mlp_set_instrument", self.h, int(on))

    def set_graphs(self, on: bool) -> None:
        """Replay the step from one CUDA graph per sync mask (captured on first use)."""
        N.call("dsx_mlp_set_graphs", self.h, int(on))

    def set_link(self, bandwidth: float, latency: float = 0.0) -> None:
        """Throttled sync link (bytes/s, s); bandwidth <= 0 disables."""
        N.call("dsx_mlp_set_link", self.h, bandwidth, latency)

    def set_overlap(self, on: bool) -> None:
        N.call("dsx_mlp_set_overlap", self.h, int(on))

    def last_step_times(self):
        out = (C.c_float * 4)()
        N.call("dsx_mlp_last_step_times", self.h, out)
        return tuple(out)

    def profile(self, reps: int = 5):
        fp = np.empty(self.L)
        bp = np.empty(self.L)
        cm = np.empty(self.L)
        N.call("dsx_mlp_profile", self.h, reps, fp.ctypes.data, bp.ctypes.data, cm.ctypes.data)
        return fp, bp, cm

    def record(self, slot: int) -> None:
        N.call("dsx_mlp_event_record", self.h, slot)

    def elapsed_ms(self, a: int, b: int) -> float:
        out = C.c_float()
        N.call("dsx_mlp_event_elapsed", self.h, a, b, C.byref(out))
        return out.value

    def launches(self) -> int:
        out = C.c_uint64()
        N.call("dsx_mlp_launch_count", self.h, C.byref(out))
        return int(out.value)


def gemm(A, B, C_out, *, M, N_, K, batch=1, a_mn=False, b_mn=False, lda, sA=0, ldb, sB=0, ldc, sC=0,
         epi=N.DSX_EPI_F32, relu=False, bias=None, s_bias=0, mask=None, ldmask=0, s_mask=0,
         accumulate=False, bn=0, dtype="bf16", stream=0, ksplit=0, s_split=0, conv=None, mask2=None) -> None:
    """dsx_gemm on torch CUDA tensors (test hook for the layer GEMMs)."""
    d = N.GemmDescC()
    d.dtype = N.DSX_BF16 if dtype == "bf16" else N.DSX_F32
    d.M, d.N, d.K, d.batch = M, N_, K, batch
    d.a_mn, d.b_mn = int(a_mn), int(b_mn)
    d.A, d.lda, d.strideA = A.data_ptr(), lda, sA
    d.B, d.ldb, d.strideB = B.data_ptr(), ldb, sB
    d.C, d.ldc, d.strideC = C_out.data_ptr(), ldc, sC
    import torch
    d.out_dtype = N.DSX_BF16 if C_out.dtype == torch.bfloat16 else N.DSX_F32
    d.epi, d.relu, d.accumulate = epi, int(relu), int(accumulate)
    d.bias = bias.data_ptr() if bias is not None else None
    d.strideBias = s_bias
    d.mask = mask.data_ptr() if mask is not None else None
    d.ldmask, d.strideMask = ldmask, s_mask
    d.bn = bn
    d.stream = stream
    d.ksplit, d.strideSplit = ksplit, s_split
    if mask2 is not None:
        d.mask2, d.ldmask2, d.strideMask2 = mask2.data_ptr(), ldmask, s_mask
    if conv is not None:  # (mode, H, W, images, cin, cout[, stride, k]): implicit-GEMM conv (input grid H x W)
        d.conv, d.conv_h, d.conv_w, d.conv_images, d.conv_cin, d.conv_cout = conv[:6]
        if len(conv) > 6:
            d.conv_stride, d.conv_k = conv[6], conv[7]
    N.call("dsx_gemm", C.byref(d))
