"""Quick A/B of the decode step: folded PPSD and AR tokens/s on the bench
workload (7B shape, E=8, prompt 128, 512 tokens), N repeats, median.
Environment knobs (PPSD_*) select kernel variants per run.

    python tools/quick_decode.py [--model 7b] [--exit 8] [--reps 3] [--eesd]
"""

import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--exit", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--eesd", action="store_true")
    ap.add_argument("--schedule", default="auto")
    args = ap.parse_args()
    config = bench.model_config(args.model)
    cfg = ppsd.PipelineConfig(config.n_layers, args.exit)
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=bench.DEEP_SCALE, deep_from=args.exit)
    prompt = bench.bench_prompt(config.vocab)
    eng = ppsd.engine_for(lm, cfg)
    eng.set_schedule(args.schedule)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("PPSD_")}, "model": args.model,
           "exit": args.exit}
    ms = []
    for _ in range(args.reps + 1):
        toks, m, _ = eng.decode(prompt, bench.NEW_TOKENS, trace=False)
        ms.append(eng.last["decode_ms"])
    out["ppsd_tok_s"] = round(bench.NEW_TOKENS / statistics.median(ms[1:]) * 1e3, 2)
    out["prefill_ms"] = eng.last.get("prefill_ms")
    out["schedule"] = eng.last["schedule"]
    out["alpha"] = m.alpha_all_measured
    ms = []
    for _ in range(args.reps + 1):
        ar = eng.decode_ar(prompt, bench.NEW_TOKENS)
        ms.append(eng.last["decode_ms"])
    out["ar_tok_s"] = round(bench.NEW_TOKENS / statistics.median(ms[1:]) * 1e3, 2)
    out["ar_equal"] = ar == toks
    if args.eesd:
        for g in bench.EESD_GAMMAS:
            ms = []
            for _ in range(2):
                et, em, _ = eng.decode_eesd(prompt, bench.NEW_TOKENS, g, trace=False)
                ms.append(eng.last["decode_ms"])
            out[f"eesd{g}_tok_s"] = round(em.committed_tokens / min(ms) * 1e3, 2)
            out[f"eesd{g}_equal"] = et[:bench.NEW_TOKENS] == toks
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
