"""Measure a Transformer layer's per-op times on the B200 (tracing.LayerTracer)
and write the hiermem TimingModel(kind="table") for a model preset, so the
reference's tracer / scheduler / simulator plan with measured B200 times.

    python tools/calibrate_timing.py --model gpt3-1.7b --update-rate 2.44e11 --out presets/b200-timing-gpt3-1.7b.json
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2303_02868_b200.tracing import LayerTracer  # noqa: E402

MODELS = {  # hiermem/presets.py:19-26
    "gpt3-1.7b": dict(seq_len=2048, d_model=2304, d_ffn=9216, num_layers=24, num_heads=24),
    "tiny-2layer": dict(seq_len=128, d_model=256, d_ffn=1024, num_layers=2, num_heads=4),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt3-1.7b", choices=sorted(MODELS))
    ap.add_argument("--update-rate", type=float, default=2.44e11, help="measured page-Adam params/s")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    m = MODELS[args.model]
    tr = LayerTracer(m["seq_len"], m["d_model"], m["d_ffn"], m["num_heads"])
    d = tr.timing_table(m["num_layers"], args.update_rate)
    d["_model"] = args.model
    Path(args.out).write_text(json.dumps(d))
    rows = d["_measured_rows"]
    print(json.dumps({"model": args.model, "rows": rows,
                      "layer_forward_s": sum(r["forward_s"] for r in rows.values()),
                      "layer_backward_s": sum(r["input_grad_s"] + r["weight_grad_s"] for r in rows.values())}))


if __name__ == "__main__":
    main()
