"""TEST INFRASTRUCTURE: the reference's toy regression problem restated in
numpy, so the drop-in can be driven through the reference's own synchronous
training loop on the GPU box (where /root/reference does not exist).

Restates hiermem/lockfree.py:45-79 (ToyTrainConfig fields used here),
:332-333 (_rng), :336-346 (init_problem), :349-356 (_teacher_forward),
:359-363 (batch_for), :366-386 (forward_backward) op for op — the same numpy
calls in the same order, so every float matches the reference's; the loss
curve it produces with the reference's own ParamBuffer/MasterState is
tests/golden/toy_sync.json (oracle/gen_golden.py:toy_sync).  Never imported
by the package.
"""
from __future__ import annotations

import math

import numpy as np


class ToyCfg:
    def __init__(self, num_layers=3, dim=16, batch_size=32, seed=5, noise_std=1.0, val_size=512):
        self.num_layers, self.dim, self.batch_size = num_layers, dim, batch_size
        self.seed, self.noise_std, self.val_size = seed, noise_std, val_size


def gen(seed: int, tag: int) -> np.random.Generator:
    return np.random.default_rng([seed, tag])


def teacher_out(teacher, readout, x, cfg: ToyCfg, noise=None):
    h = x
    for w in teacher:
        h = np.tanh(h @ w)
    y = h @ readout
    if noise is not None and cfg.noise_std > 0:
        y = y + noise.normal(0, cfg.noise_std, y.shape).astype(np.float32)
    return y.astype(np.float32)


def problem(cfg: ToyCfg):
    """(teacher, student, readout, (x_val, y_val))."""
    r = gen(cfg.seed, 0)
    d, L = cfg.dim, cfg.num_layers
    teacher = [r.normal(0, 1.0 / math.sqrt(d), (d, d)).astype(np.float32) for _ in range(L)]
    student = [r.normal(0, 0.5 / math.sqrt(d), (d, d)).astype(np.float32) for _ in range(L)]
    readout = r.normal(0, 1.0 / math.sqrt(d), (d,)).astype(np.float32)
    vr = gen(cfg.seed, 1)
    x_val = vr.normal(0, 1, (cfg.val_size, d)).astype(np.float32)
    return teacher, student, readout, (x_val, teacher_out(teacher, readout, x_val, cfg, vr))


def batch(cfg: ToyCfg, teacher, readout, it: int):
    r = gen(cfg.seed, 2 + it)
    x = r.normal(0, 1, (cfg.batch_size, cfg.dim)).astype(np.float32)
    return x, teacher_out(teacher, readout, x, cfg, r)


def loss_and_grads(ws, readout, x, y):
    """MSE of the tanh MLP and the per-layer weight gradients."""
    hs = [x]
    for w in ws:
        hs.append(np.tanh(hs[-1] @ w))
    err = hs[-1] @ readout - y
    loss = float(np.mean(err * err))
    dh = np.outer((2.0 / len(y)) * err, readout).astype(np.float32)
    grads = [None] * len(ws)
    for l in reversed(range(len(ws))):
        dz = dh * (1.0 - hs[l + 1] * hs[l + 1])
        grads[l] = (hs[l].T @ dz).astype(np.float32)
        if l > 0:
            dh = dz @ ws[l].T
    return loss, grads


def run_sync_loop(buffer, masters, cfg: ToyCfg, iterations: int, hyper, teacher, readout,
                  GradMessage, torch_io: bool = False):
    """The reference's synchronous loop body (hiermem/lockfree.py:731-769,
    DelayModel "zero": the clock terms vanish) over ANY ParamBuffer /
    MasterState pair with the reference API: read -> forward/backward ->
    accumulate in reverse -> per layer in reverse take -> update_layer ->
    record_apply -> publish(clear=False).  ``torch_io``: the buffers hold
    torch tensors (the drop-in's CUDA form); values cross to numpy for the
    toy's math only.  Returns the loss curve."""
    import torch
    L = cfg.num_layers
    curve = []
    for it in range(iterations):
        x, y = batch(cfg, teacher, readout, it)
        params = []
        for l in range(L):
            _, p16, _applied = buffer.read(l)
            p16 = p16.cpu().numpy() if torch_io else p16
            params.append(p16.astype(np.float32))
        loss, grads = loss_and_grads(params, readout, x, y)
        curve.append(loss)
        for l in reversed(range(L)):
            g16 = grads[l].astype(np.float16)
            buffer.ledger.messages_sent[l] += 1
            buffer.accumulate(GradMessage(l, torch.from_numpy(g16).cuda() if torch_io else g16, it))
        for l in reversed(range(L)):
            snap = buffer.take(l)
            if snap is None:
                continue
            grad, _count, newest = snap
            applied = masters.update_layer(l, grad, cfg.hyper)
            total = float(grad.double().sum().item()) if torch_io else float(np.sum(grad, dtype=np.float64))
            buffer.ledger.record_apply(l, total, rejected=not applied)
            p = masters.p32[l]
            buffer.publish(l, p if torch_io else p.copy(), applied_iter=newest, clear=False)
    return curve
