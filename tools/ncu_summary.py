"""Summarise an ncu --set full report into profiles/ (key metrics per kernel)
and refresh profiles/ncu_traffic.json (DRAM bytes of one adam_main launch,
read by bench.py as roofline.traffic).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_full_c2.txt "<command>" [--no-traffic]

--no-traffic: summarise only (reports of the DP kernels, whose adam_main is
the owned-page update+all-gather, must not overwrite the C2 traffic figure).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
        "nvlrx__bytes.sum", "nvltx__bytes.sum", "nvlrx__bytes_data_user.sum", "nvltx__bytes_data_user.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    args = [a for a in sys.argv[1:] if a != "--no-traffic"]
    refresh = "--no-traffic" not in sys.argv
    rep, out, cmd = args[0], Path(args[1]), args[2] if len(args) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full --clock-control none ({rep})", f"# command: {cmd}"]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        lines.append("")
        lines.append(f"Kernel Name {name}")
        vals = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {k:70s} {r[i]} {units[i]}")
                vals[k] = (r[i], units[i])
        rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
        total = float(rd[0]) * SCALE.get(rd[1], 1) + float(wr[0]) * SCALE.get(wr[1], 1)
        lines.append(f"  {'dram bytes (read+write)':70s} {total:.6g} byte")
        if "adam_main" in name:
            traffic.setdefault("adam_main", total)
    out.write_text("\n".join(lines) + "\n")
    if refresh and "adam_main" in traffic:
        tj = out.parent / "ncu_traffic.json"
        d = json.loads(tj.read_text()) if tj.exists() else {}
        d["c2:bf16"] = traffic["adam_main"]
        d["_note"] = f"dram__bytes_read.sum + dram__bytes_write.sum of one adam_main launch (bytes), {out.name}"
        tj.write_text(json.dumps(d, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
