"""C4 (T5-MoE expert-sharded pools, many small pages): K1 pack / unpack
throughput through the data-backed page manager, plus the page table size.

    python tools/pack_bench.py [--config c4] [--reps 5]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2303_02868_b200 import workloads as W  # noqa: E402
from paper_2303_02868_b200.pages import DevicePageManager  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    specs = W.config_specs(args.config)
    page = W.config_page_bytes(args.config)
    need = sum(-(-s.bytes // page) for s in specs)
    dm = DevicePageManager([("GPU", need * page, page)])
    ids = [dm.allocate(s, "GPU").tensor_id for s in specs]
    total = sum(s.bytes for s in specs)
    src = torch.randn(total // 2, device="cuda").to(torch.bfloat16).view(torch.float16)
    offs, pos = [], 0
    for s in specs:
        offs.append((pos, s.bytes // 2))
        pos += s.bytes // 2
    # warm (uploads descriptors)
    for tid, (o, n) in zip(ids, offs):
        dm.write(tid, src[o:o + n])
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    for _ in range(args.reps):
        for tid, (o, n) in zip(ids, offs):
            dm.write(tid, src[o:o + n])
    ev[1].record()
    outs = None
    for _ in range(args.reps):
        outs = [dm.read(tid) for tid in ids]
    ev[2].record()
    torch.cuda.synchronize()
    ok = all(torch.equal(o.view(torch.int16), src[a:a + n].view(torch.int16)) for o, (a, n) in zip(outs, offs))
    w_ms = ev[0].elapsed_time(ev[1]) / args.reps
    r_ms = ev[1].elapsed_time(ev[2]) / args.reps
    print(json.dumps({"config": args.config, "tensors": len(specs), "page_bytes": page,
                      "pages": dm.pools[next(iter(dm.pools))].allocated_page_count,
                      "bytes": total, "pack_ms": w_ms, "unpack_ms": r_ms,
                      "pack_gbs": 2 * total / (w_ms / 1e3) / 1e9,
                      "unpack_gbs": 2 * total / (r_ms / 1e3) / 1e9,
                      "roundtrip_bit_exact": ok,
                      "note": "GB/s counts read+write bytes; includes per-tensor host launch overhead"}))


if __name__ == "__main__":
    main()
