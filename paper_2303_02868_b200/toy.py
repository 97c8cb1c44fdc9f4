"""Demo workload for the lock-free runner: the reference's toy tanh-MLP
regression problem (hiermem/lockfree.py:45-79 ToyTrainConfig, :336-389
init_problem / batch_for / forward_backward) restated in torch on the GPU.
It only drives the update path (gradients in, published 16-bit params out);
it is not part of it.
"""
from __future__ import annotations

import math

import torch


class ToyMLP:
    def __init__(self, num_layers: int = 4, dim: int = 32, batch_size: int = 64, seed: int = 0,
                 noise_std: float = 0.01, device="cuda", grad_dtype=torch.bfloat16):
        self.L, self.dim, self.B = num_layers, dim, batch_size
        self.device = torch.device(device)
        self.noise_std = noise_std
        self.grad_dtype = grad_dtype
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        self.seed = seed
        self.teacher = [torch.randn(dim, dim, generator=g, device=self.device) / math.sqrt(dim)
                        for _ in range(num_layers)]
        self.student = [torch.randn(dim, dim, generator=g, device=self.device) * (0.5 / math.sqrt(dim))
                        for _ in range(num_layers)]
        self.readout = torch.randn(dim, generator=g, device=self.device) / math.sqrt(dim)
        self.x_val, self.y_val = self._data(10_000_019, 512)

    def _forward(self, ws, x):
        h = x
        for w in ws:
            h = torch.tanh(h @ w)
        return h @ self.readout

    def _data(self, tag: int, n: int):
        g = torch.Generator(device=self.device)
        g.manual_seed(self.seed * 1_000_003 + tag)
        x = torch.randn(n, self.dim, generator=g, device=self.device)
        y = self._forward(self.teacher, x)
        if self.noise_std > 0:
            y = y + self.noise_std * torch.randn(y.shape, generator=g, device=self.device)
        return x, y

    def batch(self, it: int):
        return self._data(2 + it, self.B)

    def loss_and_grads(self, params16, x, y):
        """MSE loss and per-layer weight gradients (forward_backward, :368-389)."""
        ws = [p.float() for p in params16]
        hs = [x]
        for w in ws:
            hs.append(torch.tanh(hs[-1] @ w))
        err = hs[-1] @ self.readout - y
        loss = (err * err).mean()
        dh = torch.outer((2.0 / len(y)) * err, self.readout)
        grads = [None] * len(ws)
        for l in reversed(range(len(ws))):
            dz = dh * (1.0 - hs[l + 1] * hs[l + 1])
            grads[l] = hs[l].T @ dz
            if l > 0:
                dh = dz @ ws[l].T
        return loss, grads

    def grads_fn(self, params16, it):
        x, y = self.batch(it)
        loss, grads = self.loss_and_grads(params16, x, y)
        return loss, torch.cat([g.reshape(-1) for g in grads]).to(self.grad_dtype)

    def val_loss(self, params16) -> float:
        return float(self.loss_and_grads(params16, self.x_val, self.y_val)[0])
