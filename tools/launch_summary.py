"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
launches, total time and share per kernel (ours vs library kernels).

    python tools/launch_summary.py gpurun_out/nb_launches.csv "<command>" > profiles/r1_launch_summary_bench.txt
"""
import csv
import sys
from collections import defaultdict


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) != len(h) or r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    ours = {k: v for k, v in tot.items() if k.startswith("hm::")}
    all_ms = sum(tot.values())
    ours_ms = sum(ours.values())
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)")
    print(f"# {cmd}")
    print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'share_all':>9s} {'ours':>4s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k[:70]:70s} {cnt[k]:8d} {tot[k]:10.3f} {tot[k] / all_ms:9.3f} {'yes' if k in ours else '':>4s}")
    print(f"# all kernels {all_ms:.3f} ms, ours {ours_ms:.3f} ms ({ours_ms / all_ms:.3f})")


if __name__ == "__main__":
    main()
