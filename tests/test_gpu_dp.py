"""Data-parallel page step on >= 2 GPUs (torchrun, NCCL): reduce-scatter of
the gradient pages, flag all-reduce, sharded page-Adam, all-gather of the
published pages — checked against the oracle in tests/dp_worker.py.
Every case runs at the largest world the box offers (2, 4 or 8 ranks: the
north star's one-box width is 8, reference tests/test_acceptance.py:188
sweeps world in {1, 2, 4, 8}); on a box with more than 2 GPUs a 2-rank
subset runs as well.  Skipped on a single-GPU box (`gpurun --gpus 2`)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


CASES = [
    (1, "bf16", "nccl", 1, 0), (2, "bf16", "nccl", 1, 0), (2, "fp16", "nccl", 1, 0),
    (2, "bf16", "p2p", 1, 0), (2, "fp16", "p2p", 1, 0), (3, "bf16", "nvls", 1, 0),
    (2, "bf16", "p2p", 3, 0), (2, "bf16", "nvls", 4, 0),
    (2, "bf16", "p2p", 3, 5),    # persistent reduce grid: 5 CTAs striding over the chunks
    (2, "bf16", "p2p", 1, "bulk1"), (2, "fp16", "p2p", 3, "bulk2"),    # bulk-copy AG epilogue
    (2, "bf16", "p2p", 3, "upd7"),    # persistent update grid (7 CTAs) + persistent reduce (5)
    (2, "bf16", "p2p", 4, "ingest"),   # host gradient streamed in per group, step starts early
    (2, "bf16", "p2p", 4, "green32"),  # reduce and update in two green contexts (SM partitions)
    (2, "bf16", "p2p", 1, "wide8"), (2, "fp16", "p2p", 3, "wide8"),  # 8-peer reduce kernel
    (2, "bf16", "p2p", 1, "ld128"),   # the 16 B-load reduce (256-bit loads are the default)
    (2, "bf16", "p2p", 1, "host"), (3, "fp16", "p2p", 1, "host"),   # fp32 state on the pinned-host tier
    (2, "bf16", "p2p", 1, "ssd"),    # fp32 state in a file per rank (SSD tier)
    (2, "bf16", "p2p", 1, "clip"), (2, "fp16", "nccl", 1, "clip"),   # global grad-norm clip over all ranks
    (2, "bf16", "p2p", 1, "onepass"), (3, "fp16", "p2p", 1, "onepass"),   # ONE fused RS+update+AG kernel
    (2, "bf16", "p2p", 1, "onepass8"),   # ... its 8-peer instantiation
    (2, "bf16", "p2p", 4, "onepass_ingest"),   # ... group by group while the host gradient arrives
    (2, "bf16", "p2p", 1, "onepass_push"), (3, "fp16", "p2p", 1, "onepass_push"),   # push form of the exchange
    (2, "bf16", "p2p", 4, "onepass_push_ingest")]
SMOKE2 = [CASES[1], CASES[3], CASES[6], CASES[12], CASES[17]]


def _world(n: int) -> int:
    return 8 if n >= 8 else 4 if n >= 4 else 2


@pytest.mark.parametrize("bucket,dtype,mode,groups,ctas", CASES)
def test_dp_step_matches_oracle(bucket, dtype, mode, groups, ctas):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    _run(_world(n), bucket, dtype, mode, groups, ctas)


@pytest.mark.parametrize("bucket,dtype,mode,groups,ctas", SMOKE2)
def test_dp_step_two_ranks(bucket, dtype, mode, groups, ctas):
    n = torch.cuda.device_count()
    if n <= 2:
        pytest.skip("the full suite above already ran at world 2")
    _run(2, bucket, dtype, mode, groups, ctas)


def _run(world, bucket, dtype, mode, groups, ctas):
    agp, upd, ingest, green, width, ld256, host = 0, 0, 0, 0, 0, 0, 0
    clip, onepass, push = 0.0, 0, 0
    if ctas == "clip":
        clip, ctas = 1.0, 0
    elif ctas in ("onepass_push", "onepass_push_ingest"):
        onepass, push, ingest, ctas = 1, 1, int(ctas.endswith("ingest")), 0
    elif ctas in ("onepass", "onepass8", "onepass_ingest"):
        onepass, width, ingest = 1, (8 if ctas == "onepass8" else 0), int(ctas == "onepass_ingest")
        ctas = 0
    elif ctas in ("host", "ssd"):
        host, ctas = (1 if ctas == "host" else "ssd"), 0
    elif ctas == "ld128":
        ld256, ctas = 1, 0
    elif ctas == "wide8":   # the 8-wide reduce instantiation (what N=8 runs), with a persistent grid when pipelined
        width, ctas = 8, 5
    elif isinstance(ctas, str) and ctas.startswith("green"):
        green, ctas = int(ctas[5:]), 0
    elif ctas == "ingest":
        ingest, ctas = 1, 0
    elif isinstance(ctas, str) and ctas.startswith("bulk"):
        agp, ctas = int(ctas[-1]), 0
    elif isinstance(ctas, str):
        upd, ctas = int(ctas[3:]), 5
    env = dict(os.environ, DP_BUCKET=str(bucket), DP_DTYPE=dtype, DP_MODE=mode, DP_GROUPS=str(groups),
               DP_REDUCE_CTAS=str(ctas), DP_AG_PUBLISH=str(agp),
               DP_UPDATE_CTAS=str(upd), DP_INGEST=str(ingest),
               DP_REDUCE_SMS=str(green), DP_REDUCE_WIDTH=str(width), DP_HOST=str(host),
               DP_CLIP=str(clip), DP_ONEPASS=str(onepass), DP_PUSH=str(push))
    visible = os.environ.get("CUDA_VISIBLE_DEVICES")
    ids = visible.split(",") if visible else [str(i) for i in range(torch.cuda.device_count())]
    env["CUDA_VISIBLE_DEVICES"] = ",".join(ids[:world])
    if ld256:
        env["DP_REDUCE_WIDE"] = "0"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29611", str(ROOT / "tests" / "dp_worker.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]


@pytest.mark.parametrize("delay", [0, 1])
def test_lockfree_runner_with_dp_step(delay):
    """Algorithm 2 on N GPUs: the lock-free runner's updating actor is the DP
    page step over the sharded pinned-host state (tests/dp_lockfree_worker.py)."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = _world(n)
    env = dict(os.environ, DP_DELAY=str(delay))
    visible = os.environ.get("CUDA_VISIBLE_DEVICES")
    ids = visible.split(",") if visible else [str(i) for i in range(n)]
    env["CUDA_VISIBLE_DEVICES"] = ",".join(ids[:world])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29612", str(ROOT / "tests" / "dp_lockfree_worker.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]


@pytest.mark.parametrize("pipe", [0, 1, 2])
def test_dp_step_full_c2_sampled(pipe):
    """The fused DP step at the size bench.py measures (C2, 4 MiB pages),
    sampled pages bit-exact (tests/dp_fullsize_worker.py)."""
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    world = _world(n)
    env = dict(os.environ, DP_PIPE=str(pipe))
    visible = os.environ.get("CUDA_VISIBLE_DEVICES")
    ids = visible.split(",") if visible else [str(i) for i in range(n)]
    env["CUDA_VISIBLE_DEVICES"] = ",".join(ids[:world])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29613", str(ROOT / "tests" / "dp_fullsize_worker.py")]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]
