"""C4 (T5-MoE expert-sharded pools, many small pages): K1 pack / unpack
throughput through the data-backed page manager, plus the page table size.

Batched: every tensor of the workload, stored back to back in one flat
buffer, is scattered into / gathered out of its pages with ONE hm_copy_runs
launch (64 KiB descriptors); per-tensor calls are timed beside it.

    python tools/pack_bench.py [--config c4] [--reps 10]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.pages import DevicePageManager, pack_many, unpack_many  # noqa: E402


def timed(fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    specs = W.config_specs(args.config)
    page = W.config_page_bytes(args.config)
    need = sum(-(-s.bytes // page) for s in specs)
    dm = DevicePageManager([("GPU", need * page, page)])
    ids = [dm.allocate(s, "GPU").tensor_id for s in specs]
    total = sum(s.bytes for s in specs)
    src = torch.randn(total // 2, device="cuda").to(torch.bfloat16)
    pack_ms, _ = timed(lambda: pack_many(dm, ids, src), args.reps)
    unpack_ms, out = timed(lambda: unpack_many(dm, ids), args.reps)
    ok = torch.equal(out, src.view(torch.uint8))
    offs, pos = [], 0
    for s in specs:
        offs.append((pos, s.bytes // 2))
        pos += s.bytes // 2
    per_tensor_ms, _ = timed(lambda: [dm.write(t, src[o:o + n]) for t, (o, n) in zip(ids, offs)], 3)
    peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
        if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0
    print(json.dumps({
        "config": args.config, "tensors": len(specs), "page_bytes": page,
        "pages": dm.pools[next(iter(dm.pools))].allocated_page_count, "bytes": total,
        "pack_ms": pack_ms, "unpack_ms": unpack_ms,
        "pack_gbs": 2 * total / (pack_ms / 1e3) / 1e9, "unpack_gbs": 2 * total / (unpack_ms / 1e3) / 1e9,
        "pack_frac_of_hbm_peak": 2 * total / (pack_ms / 1e3) / 1e9 / peak,
        "per_tensor_pack_ms": per_tensor_ms, "roundtrip_bit_exact": ok,
        "note": "GB/s counts read + write bytes; batched = one launch for all tensors"}))


if __name__ == "__main__":
    main()
