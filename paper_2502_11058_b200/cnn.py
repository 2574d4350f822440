"""Python handle over the conv-stack local step (include/dsx_nn.h dsx_cnn_*):
BASELINE configs[1]'s ResNet-18 shape as a K-worker network trained with
DreamDDP's scheduled partial synchronization.  Same vocabulary as nn.Mlp
(workers, registered layers, mask, step).

Data ("ResNet-18 on CIFAR-10-shaped synthetic data"): images N(0, 1)
[batch][32][32][3] NHWC, labels from a fixed random linear teacher over the
flattened image, one stream per (seed, worker, step) so the CPU restatement
(oracle/cnn_oracle.py) can regenerate every worker's batches.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native as N
from .nn import OPTIMIZERS

RESNET18 = dict(width=64, image=32, in_channels=3, classes=10)


def teacher(seed: int, image: int, cin: int, classes: int) -> np.ndarray:
    return np.random.default_rng([seed, 0xc1fa]).standard_normal((classes, image * image * cin)).astype(np.float32)


def batch(seed: int, worker: int, step: int, size: int, image: int, cin: int, t: np.ndarray):
    """Worker `worker`'s batch of step `step`: x ~ N(0,1) NHWC fp32, label = teacher argmax."""
    rng = np.random.default_rng([seed, worker, step, 0xc1fa])
    x = rng.standard_normal((size, image, image, cin), dtype=np.float32)
    y = np.argmax(x.reshape(size, -1).astype(np.float64) @ t.astype(np.float64).T, axis=1).astype(np.int32)
    return x, y


def init_params(seed: int, sizes, fan_in, roles) -> np.ndarray:
    """Packed parameters (layer l: W then b): He init W ~ N(0, 2/fan_in) with
    the second conv of every residual branch scaled by 1/4 (no normalisation
    layers: keeps the 8-block sum's variance bounded), head N(0, 1/fan_in),
    b = 0; all workers start from the same point."""
    rng = np.random.default_rng([seed, 0xc0de])
    parts = []
    for n, fi, role in zip(sizes, fan_in, roles):
        cout = n // (fi + 1)
        scale = np.sqrt(2.0 / fi) if role != "head" else np.sqrt(1.0 / fi)
        if role == "b":
            scale *= 0.25
        parts.append((rng.standard_normal(cout * fi) * scale).astype(np.float32))
        parts.append(np.zeros(cout, dtype=np.float32))
    return np.concatenate(parts)


def conv_geometry(width: int, image: int):
    """(Cin, Cout, k, Ho) of every conv in registration order (dsx_cnn_create)."""
    out = [(8, width, 3, image)]
    cin, H = width, image
    for s in range(4):
        w = width << s
        for blk in range(2):
            stride = 2 if (s > 0 and blk == 0) else 1
            Ho = (H - 1) // stride + 1
            out += [(cin, w, 3, Ho), (w, w, 3, Ho)]
            if stride != 1 or cin != w:
                out.append((cin, w, 1, Ho))
            cin, H = w, Ho
    return out


def conv_stack_flops(width: int, image: int, classes: int, batch: int) -> float:
    f = 0.0
    for i, (cin, cout, k, Ho) in enumerate(conv_geometry(width, image)):
        f += 2.0 * batch * Ho * Ho * cout * k * k * cin * (2 if i == 0 else 3)
    return f + 3 * 2.0 * batch * (width << 3) * classes


class Cnn:
    """K (or K/N per rank) device-resident conv-stack workers."""

    def __init__(self, batch_size: int, workers_total: int, workers_local: int | None = None,
                 worker_begin: int = 0, width: int = 64, image: int = 32, in_channels: int = 3,
                 classes: int = 10, dtype: str = "bf16", optimizer: str = "momentum", momentum: float = 0.9,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0,
                 device: int = 0):
        self.batch = int(batch_size)
        self.K = workers_total
        self.kl = workers_local if workers_local is not None else workers_total
        self.width, self.image, self.cin, self.classes = width, image, in_channels, classes
        self.dtype = dtype
        d = N.CnnDescC()
        d.device = device
        d.dtype = N.DSX_BF16 if dtype == "bf16" else N.DSX_F32
        d.workers_total = workers_total
        d.worker_begin = worker_begin
        d.workers_local = self.kl
        d.width, d.image, d.in_channels, d.classes = width, image, in_channels, classes
        d.batch = self.batch
        d.optimizer = OPTIMIZERS[optimizer]
        d.momentum, d.beta1, d.beta2, d.eps, d.weight_decay = momentum, beta1, beta2, eps, weight_decay
        h = C.c_void_p()
        N.call("dsx_cnn_create", C.byref(d), C.byref(h))
        self.h = h
        layers = C.c_int()
        total = C.c_uint64()
        N.call("dsx_cnn_param_layout", self.h, C.byref(layers), C.byref(total), None, None)
        self.L = int(layers.value)
        offs = (C.c_uint64 * (self.L + 1))()
        fan = (C.c_int * self.L)()
        N.call("dsx_cnn_param_layout", self.h, None, None, offs, fan)
        self.P = int(total.value)
        self.offsets = [int(x) for x in offs]
        self.fan_in = [int(x) for x in fan]
        self._keep = None

    def layer_sizes(self):
        return [b - a for a, b in zip(self.offsets[:-1], self.offsets[1:])]

    def close(self):
        if getattr(self, "h", None):
            N.load_dsx().dsx_cnn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_params(self, local: int, flat: np.ndarray) -> None:
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        assert flat.size == self.P
        N.call("dsx_cnn_set_params", self.h, local, flat.ctypes.data)

    def get_params(self, local: int) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        N.call("dsx_cnn_get_params", self.h, local, out.ctypes.data)
        return out

    def set_batch(self, x: np.ndarray, labels: np.ndarray) -> None:
        """Host batch [kl][batch][image][image][cin] fp32 + labels [kl][batch]."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        y = np.ascontiguousarray(labels, dtype=np.int32)
        self._keep = (x, y)
        N.call("dsx_cnn_set_batch", self.h, x.ctypes.data, y.ctypes.data, 0)

    def set_batch_ptr(self, x_ptr: int, labels_ptr: int, on_device: bool) -> None:
        N.call("dsx_cnn_set_batch", self.h, C.c_void_p(x_ptr), C.c_void_p(labels_ptr), int(on_device))

    def step(self, lr: float, t: int, mask) -> None:
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        N.call("dsx_cnn_step", self.h, lr, t, mask.ctypes.data)

    def last_loss(self) -> np.ndarray:
        out = np.empty(self.kl, dtype=np.float32)
        N.call("dsx_cnn_last_loss", self.h, out.ctypes.data)
        return out

    def sync(self) -> None:
        N.call("dsx_cnn_sync", self.h)

    def comm_init(self, uid: bytes, nranks: int, rank: int) -> None:
        buf = C.create_string_buffer(uid, 128)
        N.call("dsx_cnn_comm_init", self.h, buf, nranks, rank)

    def set_instrument(self, on: bool) -> None:
        N.call("dsx_cnn_set_instrument", self.h, int(on))

    def last_step_times(self):
        out = (C.c_float * 4)()
        N.call("dsx_cnn_last_step_times", self.h, out)
        return tuple(out)

    def profile(self, reps: int = 5):
        """Per-layer FP / BP / average seconds (dsx_cnn_profile)."""
        fp, bp, cm = (np.empty(self.L) for _ in range(3))
        N.call("dsx_cnn_profile", self.h, reps, fp.ctypes.data, bp.ctypes.data, cm.ctypes.data)
        return fp, bp, cm

    def flops_per_worker(self) -> float:
        """GEMM flops of one local step: forward, wgrad and dgrad (none into the stem's input)."""
        return conv_stack_flops(self.width, self.image, self.classes, self.batch)

    def set_link(self, bandwidth: float, latency: float = 0.0) -> None:
        """Throttled sync link (bytes/s, s); bandwidth <= 0 disables."""
        N.call("dsx_cnn_set_link", self.h, bandwidth, latency)

    def set_overlap(self, on: bool) -> None:
        N.call("dsx_cnn_set_overlap", self.h, int(on))

    def record(self, slot: int) -> None:
        N.call("dsx_cnn_event_record", self.h, slot)

    def elapsed_ms(self, a: int, b: int) -> float:
        out = C.c_float()
        N.call("dsx_cnn_event_elapsed", self.h, a, b, C.byref(out))
        return out.value

    def launches(self) -> int:
        out = C.c_uint64()
        N.call("dsx_cnn_launch_count", self.h, C.byref(out))
        return int(out.value)
