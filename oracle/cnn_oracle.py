"""CPU restatement of the conv-stack local step (BASELINE configs[1], the
ResNet-18 shape) + scheduled partial sync (TEST INFRASTRUCTURE ONLY: imported
by tests/ and bench.py's checker, never by the product path).

Parity status: **unpinned by the reference** (the reference has no neural
network — SPEC.md:8, SURVEY §8c row "NN models"); like oracle/mlp_oracle.py
this restates the reference's plsgd_step structure (trainer.cpp:187-235) with
the network's gradient in place of the quadratic's, in float64:
  * every worker takes its local step (FP -> softmax cross-entropy -> BP in
    the order head, blocks last to first (shortcut, conv b, conv a), stem;
    each layer's optimizer right after its gradient, with the pre-update
    weights feeding the input gradient);
  * masked registered layers are replaced by pairwise_coord_sum(...)/K
    (trainer.cpp:31-38), optimizer states stay local.
The network is the one include/dsx_nn.h documents for dsx_cnn: 3x3 stem on
the input zero-padded to 8 channels, 4 stages x 2 basic blocks (widths
w0 << s; stride 2 + 1x1 projection shortcut entering stages 1-3), global
average pool, linear head; NHWC activations, W [Cout][kh][kw][Cin].
"""
from __future__ import annotations

import numpy as np

from .mlp_oracle import pairwise_sum


def topology(width, image, cin_pad=8, classes=10):
    """Registered layers in forward order: dicts (cin, cout, k, stride, H, relu, role)."""
    convs = [dict(cin=cin_pad, cout=width, k=3, stride=1, H=image, relu=True, role="stem")]
    blocks = []
    cin, H = width, image
    for s in range(4):
        w = width << s
        for blk in range(2):
            stride = 2 if (s > 0 and blk == 0) else 1
            Ho = (H + 2 - 3) // stride + 1
            a = len(convs)
            convs.append(dict(cin=cin, cout=w, k=3, stride=stride, H=H, relu=True, role="a"))
            convs.append(dict(cin=w, cout=w, k=3, stride=1, H=Ho, relu=False, role="b"))
            sc = -1
            if stride != 1 or cin != w:
                sc = len(convs)
                convs.append(dict(cin=cin, cout=w, k=1, stride=stride, H=H, relu=False, role="sc"))
            blocks.append((a, a + 1, sc))
            cin, H = w, Ho
    head = dict(cin=cin, cout=classes, role="head")
    return convs, blocks, head


def layer_sizes(width, image, cin_pad=8, classes=10):
    convs, _, head = topology(width, image, cin_pad, classes)
    return [c["cout"] * c["k"] * c["k"] * c["cin"] + c["cout"] for c in convs] + \
        [head["cout"] * head["cin"] + head["cout"]]


def _pad(c):
    return 1 if c["k"] == 3 else 0


def im2col(x, c):
    """x [B][H][W][C] -> col [B][Ho][Wo][k][k][C] (zero outside the image)."""
    k, s, p = c["k"], c["stride"], _pad(c)
    B, H, W, C = x.shape
    Ho = (H + 2 * p - k) // s + 1
    xp = np.zeros((B, H + 2 * p, W + 2 * p, C), dtype=x.dtype)
    xp[:, p:p + H, p:p + W] = x
    col = np.empty((B, Ho, Ho, k, k, C), dtype=x.dtype)
    for kh in range(k):
        for kw in range(k):
            col[:, :, :, kh, kw] = xp[:, kh:kh + s * Ho:s, kw:kw + s * Ho:s]
    return col


def col2im(dcol, c, H):
    """Adjoint of im2col: dcol [B][Ho][Wo][k][k][C] -> dx [B][H][W][C]."""
    k, s, p = c["k"], c["stride"], _pad(c)
    B, Ho = dcol.shape[0], dcol.shape[1]
    C = dcol.shape[-1]
    dxp = np.zeros((B, H + 2 * p, H + 2 * p, C), dtype=dcol.dtype)
    for kh in range(k):
        for kw in range(k):
            dxp[:, kh:kh + s * Ho:s, kw:kw + s * Ho:s] += dcol[:, :, :, kh, kw]
    return dxp[:, p:p + H, p:p + H]


class CnnOracle:
    def __init__(self, width, image, in_channels, classes, init, workers, optimizer="momentum", momentum=0.9,
                 beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, dtype=np.float64):
        self.dtype = dtype
        self.image, self.cin, self.classes = image, in_channels, classes
        self.convs, self.blocks, self.head = topology(width, image, 8, classes)
        self.K = workers
        self.opt = optimizer
        self.mu, self.b1, self.b2, self.eps, self.wd = momentum, beta1, beta2, eps, weight_decay
        sizes = layer_sizes(width, image, 8, classes)
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.w = [np.asarray(init, dtype=dtype).copy() for _ in range(workers)]
        self.m = [np.zeros_like(self.w[0]) for _ in range(workers)]
        self.v = [np.zeros_like(self.w[0]) for _ in range(workers)]
        self.loss = np.zeros(workers)

    def _wb(self, k, l, cout, kc):
        lo = self.offsets[l]
        return self.w[k][lo:lo + cout * kc].reshape(cout, kc), self.w[k][lo + cout * kc:self.offsets[l + 1]]

    def _update(self, k, l, g, lr, t):
        lo, hi = self.offsets[l], self.offsets[l + 1]
        w, m, v = self.w[k], self.m[k], self.v[k]
        if self.opt == "sgd":
            w[lo:hi] -= lr * (g + self.wd * w[lo:hi])
        elif self.opt == "momentum":
            m[lo:hi] = self.mu * m[lo:hi] + g + self.wd * w[lo:hi]
            w[lo:hi] -= lr * m[lo:hi]
        else:
            m[lo:hi] = self.b1 * m[lo:hi] + (1 - self.b1) * g
            v[lo:hi] = self.b2 * v[lo:hi] + (1 - self.b2) * g * g
            bc1, bc2 = 1 - self.b1 ** (t + 1), 1 - self.b2 ** (t + 1)
            w[lo:hi] -= lr * ((m[lo:hi] / bc1) / (np.sqrt(v[lo:hi] / bc2) + self.eps) + self.wd * w[lo:hi])

    def _conv(self, k, l, x):
        c = self.convs[l]
        kc = c["k"] * c["k"] * c["cin"]
        W, b = self._wb(k, l, c["cout"], kc)
        col = im2col(x, c)
        z = col.reshape(-1, kc) @ W.T + b
        y = z.reshape(col.shape[:3] + (c["cout"],))
        return (np.maximum(y, 0.0) if c["relu"] else y), col

    def _conv_back(self, k, l, g, col, lr, t, dgrad=True):
        """g = dL/d(conv output) [B][Ho][Wo][Cout] -> update; returns dcol or None."""
        c = self.convs[l]
        kc = c["k"] * c["k"] * c["cin"]
        W, _ = self._wb(k, l, c["cout"], kc)
        g2 = g.reshape(-1, c["cout"])
        dW = g2.T @ col.reshape(-1, kc)
        db = g2.sum(axis=0)
        dcol = (g2 @ W).reshape(col.shape) if dgrad else None
        self._update(k, l, np.concatenate([dW.ravel(), db]), lr, t)
        return dcol

    def local_step(self, k, x, y, lr, t):
        B = x.shape[0]
        x0 = np.zeros((B, self.image, self.image, 8), dtype=self.dtype)
        x0[..., :self.cin] = x
        stem, stem_col = self._conv(k, 0, x0)
        h = stem
        saved = []
        for (a, b, sc) in self.blocks:
            ya, ca = self._conv(k, a, h)
            yb, cb = self._conv(k, b, ya)
            if sc >= 0:
                ys, cs = self._conv(k, sc, h)
            else:
                ys, cs = h, None
            out = np.maximum(yb + ys, 0.0)
            saved.append((h, ya, ca, cb, cs, out))
            h = out
        C = h.shape[-1]
        pool = h.reshape(B, -1, C).mean(axis=1)
        hl = len(self.convs)
        Wh = self.w[k][self.offsets[hl]:self.offsets[hl] + self.classes * C].reshape(self.classes, C)
        bh = self.w[k][self.offsets[hl] + self.classes * C:self.offsets[hl + 1]]
        z = pool @ Wh.T + bh
        zmax = z.max(axis=1, keepdims=True)
        lse = zmax[:, 0] + np.log(np.exp(z - zmax).sum(axis=1))
        self.loss[k] = float(np.mean(lse - z[np.arange(B), y]))
        p = np.exp(z - lse[:, None])
        p[np.arange(B), y] -= 1.0
        dz = p / B
        dW = dz.T @ pool
        db = dz.sum(axis=0)
        dpool = dz @ Wh
        self._update(k, hl, np.concatenate([dW.ravel(), db]), lr, t)
        HW = h.shape[1] * h.shape[2]
        gy = np.broadcast_to((dpool / HW)[:, None, None, :], h.shape).copy()
        for bi in range(len(self.blocks) - 1, -1, -1):
            a, b, sc = self.blocks[bi]
            hin, ya, ca, cb, cs, out = saved[bi]
            ga = gy * (out > 0)
            if sc >= 0:
                dcs = self._conv_back(k, sc, ga, cs, lr, t)
                gsc = col2im(dcs, self.convs[sc], hin.shape[1])
            else:
                gsc = ga
            dcb = self._conv_back(k, b, ga, cb, lr, t)
            gh = col2im(dcb, self.convs[b], ya.shape[1]) * (ya > 0)
            dca = self._conv_back(k, a, gh, ca, lr, t)
            gy = col2im(dca, self.convs[a], hin.shape[1]) + gsc
        self._conv_back(k, 0, gy * (stem > 0), stem_col, lr, t, dgrad=False)

    def step(self, batches, lr, t, mask):
        """One plsgd_step: batches[k] = (x [B][H][W][Cin], y [B]); mask[L+1], 1-based."""
        for k in range(self.K):
            self.local_step(k, np.asarray(batches[k][0], dtype=self.dtype), batches[k][1], lr, t)
        for l in range(1, len(self.offsets)):
            if not mask[l]:
                continue
            lo, hi = self.offsets[l - 1], self.offsets[l]
            mean = pairwise_sum([w[lo:hi] for w in self.w], 0, self.K) / self.K
            for w in self.w:
                w[lo:hi] = mean
