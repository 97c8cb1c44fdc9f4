"""Tracer hooks on real torch ops: measured production times for the
reference's planning stack.

The reference derives tensor lifetimes on the logical timeline of
hiermem/tracer.py:1-32 and charges production times from a TimingModel
(:84-129) — proportional to bytes by default; ``kind="table"`` takes a
measured ``name -> (cpu_time, gpu_time)`` table.  The paper measures them
with hooks around each op ("time.time() / CudaEvent").
``LayerTracer`` runs the twelve Table-1 ops of one Transformer layer
(hiermem/footprint.py:105-122) in bf16 on the GPU, times forward and
backward of each with CUDA events, and emits that table for the tensor
inventory names (footprint.py:184-219):

* ``*.act16``  gpu_time = forward + input-gradient time of the op (the
  simulator charges half at the forward op and half at the backward op,
  hiermem/simengine.py:6-9);
* ``*.grad16`` gpu_time = the weight-gradient part of the backward op;
* ``*.param16`` cpu_time = the page-Adam update time of the tensor at a
  measured update rate (params/s) — on this system the optimizer runs on
  the GPU, so it is the GPU update time in the reference's update slot.
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as F

ROWS = ("attn.linear_qkv", "attn.matmul_scores", "attn.scaled_mask_softmax", "attn.matmul_context",
        "attn.linear_out", "post_attn.add", "post_attn.layer_norm", "ffn.linear_in", "ffn.gelu",
        "ffn.linear_out", "post_ffn.add", "post_ffn.layer_norm")
PARAM_ROWS = {"attn.linear_qkv", "attn.linear_out", "post_attn.layer_norm", "ffn.linear_in",
              "ffn.linear_out", "post_ffn.layer_norm"}


class LayerTracer:
    def __init__(self, seq_len: int, d_model: int, d_ffn: int, num_heads: int, batch_size: int = 1,
                 device="cuda", dtype=torch.bfloat16):
        self.s, self.d, self.f, self.h, self.b = seq_len, d_model, d_ffn, num_heads, batch_size
        self.dev, self.dt = torch.device(device), dtype

    def _ops(self):
        b, s, d, f, h = self.b, self.s, self.d, self.f, self.h
        dh = d // h
        kw = dict(device=self.dev, dtype=self.dt)
        x = torch.randn(b * s, d, **kw)
        wqkv = torch.randn(d, 3 * d, **kw) / math.sqrt(d)
        wo = torch.randn(d, d, **kw) / math.sqrt(d)
        w1 = torch.randn(d, f, **kw) / math.sqrt(d)
        w2 = torch.randn(f, d, **kw) / math.sqrt(f)
        ln_w, ln_b = torch.ones(d, **kw), torch.zeros(d, **kw)
        q = torch.randn(b * h, s, dh, **kw)
        k = torch.randn(b * h, s, dh, **kw)
        scores = torch.randn(b * h, s, s, **kw)
        probs = torch.softmax(scores.float(), -1).to(self.dt)
        v = torch.randn(b * h, s, dh, **kw)
        hid = torch.randn(b * s, f, **kw)
        mask = torch.ones(s, s, device=self.dev, dtype=torch.bool).tril()
        # (row, inputs that need grad, params among them, fn)
        return {
            "attn.linear_qkv": ([x, wqkv], {1}, lambda a, w: a @ w),
            "attn.matmul_scores": ([q, k], set(), lambda a, c: a @ c.transpose(1, 2) / math.sqrt(dh)),
            "attn.scaled_mask_softmax": ([scores], set(),
                                         lambda z: torch.softmax(z.masked_fill(~mask, -1e4), -1)),
            "attn.matmul_context": ([probs, v], set(), lambda p_, v_: p_ @ v_),
            "attn.linear_out": ([x, wo], {1}, lambda a, w: a @ w),
            "post_attn.add": ([x, x.clone()], set(), lambda a, c: a + c),
            "post_attn.layer_norm": ([x, ln_w, ln_b], {1, 2}, lambda a, w, bb: F.layer_norm(a, (d,), w, bb)),
            "ffn.linear_in": ([x, w1], {1}, lambda a, w: a @ w),
            "ffn.gelu": ([hid], set(), F.gelu),
            "ffn.linear_out": ([hid, w2], {1}, lambda a, w: a @ w),
            "post_ffn.add": ([x, x.clone()], set(), lambda a, c: a + c),
            "post_ffn.layer_norm": ([x, ln_w, ln_b], {1, 2}, lambda a, w, bb: F.layer_norm(a, (d,), w, bb)),
        }

    @staticmethod
    def _time(fn, reps):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3 / reps

    def measure(self, reps: int = 10) -> dict[str, dict[str, float]]:
        """Per row: forward, input-gradient and weight-gradient seconds."""
        out = {}
        for row, (inputs, params, fn) in self._ops().items():
            ins = [t.detach().requires_grad_(True) for t in inputs]
            y = fn(*ins)
            gy = torch.randn_like(y)
            fwd = self._time(lambda: fn(*ins), reps)
            acts = [t for i, t in enumerate(ins) if i not in params]
            pars = [t for i, t in enumerate(ins) if i in params]

            def grad_of(ts):
                return lambda: torch.autograd.grad(fn(*ins), ts, gy, allow_unused=True)

            dx = self._time(grad_of(acts), reps) - fwd if acts else 0.0
            dw = self._time(grad_of(pars), reps) - fwd if pars else 0.0
            out[row] = {"forward_s": fwd, "input_grad_s": max(dx, 0.0), "weight_grad_s": max(dw, 0.0)}
        return out

    def timing_table(self, num_layers: int, update_params_per_s: float, reps: int = 10) -> dict:
        """hiermem TimingModel(kind="table") dict for the inventory of a
        TransformerConfig with this layer shape and ``num_layers`` layers."""
        m = self.measure(reps)
        d, f = self.d, self.f
        param_elems = {"attn.linear_qkv": 3 * d * d, "attn.linear_out": d * d, "post_attn.layer_norm": d,
                       "ffn.linear_in": d * f, "ffn.linear_out": d * f, "post_ffn.layer_norm": d}
        table = {}
        for layer in range(num_layers):
            for row in ROWS:
                base = f"L{layer}.{row}"
                r = m[row]
                table[f"{base}.act16"] = [0.0, r["forward_s"] + r["input_grad_s"]]
                if row in PARAM_ROWS:
                    table[f"{base}.grad16"] = [0.0, r["weight_grad_s"]]
                    table[f"{base}.param16"] = [param_elems[row] / update_params_per_s, 0.0]
                    table[f"{base}.optim32"] = [0.0, 0.0]
        return {"kind": "table", "table": table, "_measured_rows": m}
