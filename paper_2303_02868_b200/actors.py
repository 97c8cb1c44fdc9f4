"""Lock-free delayed update (Angel-PTM Algorithm 2) on CUDA streams.

The reference runs three actors — GPU, buffering, updating — as coroutines
on a virtual clock or as threads (hiermem/lockfree.py:403-526, 542-640):
the GPU actor computes against whatever parameters are published, the
buffering actor accumulates gradients and hands them over (clear at take),
the updating actor sweeps layers in reverse (take -> fetch -> update ->
publish -> store).  Here the actors are streams:

* compute stream  (GPU actor): forward/backward against a published 16-bit
  page buffer, then ``accumulate_flat`` of the gradient into the active
  gradient page buffer (the buffering actor's accumulate, K3);
* update stream   (updating actor): ``sweep`` — or ``swap_sweep`` when the
  fp32 state lives in pinned host memory, or the data-parallel page step
  (reduce-scatter -> update -> all-gather) — takes the buffer, updates and
  publishes into the inactive parameter buffer (K2 + K8);
* events replace mailboxes: the update of iteration k waits for the
  accumulate of k; with ``delay=1`` the compute of k+1 reads the parameters
  published by the update of k-1 and runs concurrently with the update of k
  (bounded staleness 1, the pipelined steady state of the reference's
  lock-free mode); ``delay=0`` is the synchronous baseline (run_sync,
  lockfree.py:719-771) where every iteration waits for the previous update.

Double buffering is race-free by construction: the update of k writes the
parameter buffer that iteration k read (it starts after k's accumulate,
which follows k's reads on the compute stream), and iteration k+1
accumulates into the gradient buffer taken by the update of k-1, which it
already waits for (its parameters come from that update).  Host bookkeeping
(pending counts, versions, staleness, ledger counts) follows enqueue order.
"""
from __future__ import annotations

import time
from collections import Counter
from dataclasses import dataclass, field

import torch

from .errors import ConfigError
from .lockfree import ParamBuffer, sweep


@dataclass
class RunReport:
    mode: str
    iterations: int
    loss_curve: list = field(default_factory=list)
    staleness_histogram: dict = field(default_factory=dict)
    max_staleness: int = 0
    wall_s: float = 0.0
    iter_ms: float = 0.0
    publishes: int = 0
    rejected_updates: int = 0


class LockFreeRunner:
    def __init__(self, buffer: ParamBuffer, masters, hyper, *, delay: int = 1,
                 compute_stream=None, update_stream=None, update=None):
        if delay not in (0, 1):
            raise ConfigError("delay must be 0 (synchronous) or 1 (lock-free, staleness <= 1)")
        self.buffer, self.masters, self.hyper, self.delay = buffer, masters, hyper, delay
        dev = buffer.device
        self.cs = compute_stream or torch.cuda.Stream(dev)
        self.us = update_stream or torch.cuda.Stream(dev)
        from .swap import HostMasterState, swap_sweep
        # the updating actor's step: the fused sweep, the swap sweep for a
        # host-tier state, or a caller's (e.g. the data-parallel page step,
        # ``lambda buf, ms, hyper, stream: dp.step(hyper, stream=stream)``)
        self._sweep = update or (swap_sweep if isinstance(masters, HostMasterState) else sweep)
        self._pub: list[tuple[torch.cuda.Event, int, int]] = []   # (event, psel, version)
        self._it = 0                  # global iteration counter across run() calls
        self._psel0 = buffer._psel[0]
        if any(p != self._psel0 for p in buffer._psel):
            raise ConfigError("all layers must start in the same published buffer")

    def params(self, it: int):
        """Per-layer 16-bit parameter tensors the GPU actor reads at iteration
        ``it`` (zero-copy views of the published pages where contiguous)."""
        src = it - 1 - self.delay
        if src >= 0:
            ev, psel, _ = self._pub[src]
            self.cs.wait_event(ev)
        else:
            psel = self._psel0
        views = [self.buffer.layer_view(l, psel, stream=self.cs) for l in range(self.buffer.num_layers)]
        return views, src

    def run(self, iterations: int, grads_fn, mode: str = "lockfree") -> RunReport:
        """``grads_fn(params, it) -> (loss_tensor, flat_grad)``, enqueued on the
        compute stream; ``flat_grad`` holds every layer's gradient in order."""
        rep = RunReport(mode=mode, iterations=iterations)
        stale = Counter()
        losses = []
        torch.cuda.synchronize(self.buffer.device)
        t0 = time.perf_counter()
        for _ in range(iterations):
            it = self._it
            self._it += 1
            with torch.cuda.stream(self.cs):
                params, src = self.params(it)
                applied = -1 if src < 0 else src
                stale[max(0, (it - 1) - applied)] += self.buffer.num_layers
                loss, flat = grads_fn(params, it)
                losses.append(loss)
                self.buffer.accumulate_flat(flat, it, stream=self.cs)
                acc = torch.cuda.Event()
                acc.record(self.cs)
            self.us.wait_event(acc)
            with torch.cuda.stream(self.us):
                self._sweep(self.buffer, self.masters, self.hyper, stream=self.us)
                pub = torch.cuda.Event()
                pub.record(self.us)
            self._pub.append((pub, self.buffer._psel[0], self.buffer._version[0]))
            rep.publishes += self.buffer.num_layers
        torch.cuda.synchronize(self.buffer.device)
        rep.wall_s = time.perf_counter() - t0
        rep.iter_ms = rep.wall_s * 1e3 / iterations
        rep.loss_curve = [float(l) for l in torch.stack(losses).cpu().tolist()]
        rep.staleness_histogram = dict(stale)
        rep.max_staleness = max(stale) if stale else 0
        return rep
