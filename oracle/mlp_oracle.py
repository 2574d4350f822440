"""CPU restatement of the NN local step + scheduled partial sync (TEST
INFRASTRUCTURE ONLY: imported by tests/ and bench.py's checker, never by the
product path).

Parity status: **unpinned by the reference.**  The reference has no neural
network (SPEC.md:8 lists "training actual GPT-2/Llama/ResNet models ...
Adam/momentum preconditioner state" as out of scope; SURVEY §8c row "NN
models"), so there are no golden vectors to pin against.  This file restates
the reference's step structure with the NN gradient in place of the
quadratic's, in float64:
  * plsgd_step (trainer.cpp:187-235): every worker takes its local step
    (here FP -> softmax cross-entropy -> BP, each layer's optimizer update
    right after its gradient), then the masked blocks (registered layers) are
    replaced by the cross-worker mean;
  * the mean is pairwise_coord_sum(...)/K (trainer.cpp:31-38): split at
    lo + n/2, which for K in {1,2,4,8} is also the device kernels' order;
  * masks come from the same sync_mask helper (trainer.cpp:202-224);
  * optimizer states are per worker and never averaged (Alg. 1 averages
    parameters only).
"""
from __future__ import annotations

import numpy as np


def pairwise_sum(rows, lo, n):
    """pairwise_coord_sum (trainer.cpp:31-38) over whole vectors."""
    if n == 1:
        return rows[lo]
    if n == 2:
        return rows[lo] + rows[lo + 1]
    h = n // 2
    return pairwise_sum(rows, lo, h) + pairwise_sum(rows, lo + h, n - h)


def split(flat, widths):
    """Packed vector -> [(W[out][in], b[out])] views."""
    out, o = [], 0
    for i, n in zip(widths[:-1], widths[1:]):
        W = flat[o:o + i * n].reshape(n, i)
        o += i * n
        b = flat[o:o + n]
        o += n
        out.append((W, b))
    return out


class MlpOracle:
    def __init__(self, widths, init, workers, optimizer="momentum", momentum=0.9, beta1=0.9, beta2=0.999,
                 eps=1e-8, weight_decay=0.0, dtype=np.float64):
        self.dtype = dtype  # float64 (the checker); float32 only to measure rounding sensitivity
        self.widths = list(widths)
        self.K = workers
        self.opt = optimizer
        self.mu, self.b1, self.b2, self.eps, self.wd = momentum, beta1, beta2, eps, weight_decay
        self.w = [np.asarray(init, dtype=dtype).copy() for _ in range(workers)]
        self.m = [np.zeros_like(self.w[0]) for _ in range(workers)]
        self.v = [np.zeros_like(self.w[0]) for _ in range(workers)]
        self.offsets = [0]
        for i, n in zip(self.widths[:-1], self.widths[1:]):
            self.offsets.append(self.offsets[-1] + i * n + n)
        self.loss = np.zeros(workers)

    def _update(self, k, lo, hi, g, lr, t):
        w, m, v = self.w[k], self.m[k], self.v[k]
        if self.opt == "sgd":
            g = g + self.wd * w[lo:hi]
            w[lo:hi] -= lr * g
        elif self.opt == "momentum":
            g = g + self.wd * w[lo:hi]
            m[lo:hi] = self.mu * m[lo:hi] + g
            w[lo:hi] -= lr * m[lo:hi]
        else:
            m[lo:hi] = self.b1 * m[lo:hi] + (1 - self.b1) * g
            v[lo:hi] = self.b2 * v[lo:hi] + (1 - self.b2) * g * g
            bc1, bc2 = 1 - self.b1 ** (t + 1), 1 - self.b2 ** (t + 1)
            w[lo:hi] -= lr * ((m[lo:hi] / bc1) / (np.sqrt(v[lo:hi] / bc2) + self.eps) + self.wd * w[lo:hi])

    def local_step(self, k, x, y, lr, t):
        L = len(self.widths) - 1
        layers = split(self.w[k], self.widths)
        acts = [np.asarray(x, dtype=self.dtype)]
        for l, (W, b) in enumerate(layers):
            z = acts[-1] @ W.T + b
            acts.append(np.maximum(z, 0.0) if l < L - 1 else z)
        z = acts[-1]
        zmax = z.max(axis=1, keepdims=True)
        lse = zmax[:, 0] + np.log(np.exp(z - zmax).sum(axis=1))
        B = z.shape[0]
        self.loss[k] = float(np.mean(lse - z[np.arange(B), y]))
        p = np.exp(z - lse[:, None])
        p[np.arange(B), y] -= 1.0
        dz = p / B
        for l in range(L - 1, -1, -1):
            W, b = split(self.w[k], self.widths)[l]
            a = acts[l]
            dW = dz.T @ a
            db = dz.sum(axis=0)
            dprev = (dz @ W) * (a > 0) if l > 0 else None
            lo, hi = self.offsets[l], self.offsets[l + 1]
            self._update(k, lo, hi, np.concatenate([dW.ravel(), db]), lr, t)
            dz = dprev

    def step(self, batches, lr, t, mask):
        """One plsgd_step: batches[k] = (x, y); mask[L+1], 1-based."""
        for k in range(self.K):
            self.local_step(k, batches[k][0], batches[k][1], lr, t)
        for l in range(1, len(self.widths)):
            if not mask[l]:
                continue
            lo, hi = self.offsets[l - 1], self.offsets[l]
            mean = pairwise_sum([w[lo:hi] for w in self.w], 0, self.K) / self.K
            for w in self.w:
                w[lo:hi] = mean
