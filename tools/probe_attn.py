"""Decode-attention latency per launch (attn_core.cuh split-K kernel) at the
7B shape (32 kv heads, hd 128, bf16 KV): n_vec query vectors in one group,
longest context ctx, back-to-back launches walking the layers.

    python tools/probe_attn.py [--model 7b] [--out profiles/r02_attn_probe.json]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200.decode import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    base = {"7b": ppsd.TransformerConfig.llama2_7b, "13b": ppsd.TransformerConfig.llama2_13b,
            "70b": ppsd.TransformerConfig.llama2_70b}[args.model](max_ctx=1024)
    import dataclasses

    config = dataclasses.replace(base, n_layers=args.layers)
    lm = ppsd.TransformerLM(config, seed=0)
    cfg = ppsd.PipelineConfig(args.layers, 1)
    rows = []
    mode = os.environ.get("PPSD_ATTN_CLB", "cluster")
    if True:
        eng = Engine(lm.model_desc(), lm.weights_struct(), cfg, device=lm.device.index)
        for nv in (1, 4, 11):
            for ctx in (128, 384, 640, 1000):
                ms, b = eng.probe_attn(nv, ctx, 200)
                rows.append(dict(kernel=mode, n_vec=nv, ctx=ctx, us=round(ms * 1e3, 3),
                                 gbs=round(b / (ms / 1e3) / 1e9, 1)))
                print(json.dumps(rows[-1]), flush=True)
        eng.close()
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(dict(model=args.model, rows=rows), fh, indent=1)


if __name__ == "__main__":
    main()
