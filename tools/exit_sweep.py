"""BASELINE config 5: exit-position sweep E in {4, 8, 12, 16} on the Llama-2-7B
shape — PPSD vs vanilla EESD (gamma 5, 10) vs autoregressive, measured
acceptance and speedup, next to the paper's closed forms (Eq. 5 / Eq. 7).

One B200, bs=1, prompt 128, 512 new tokens, decode phase timed with CUDA
events (prefill excluded). deep_scale is held fixed and deep_from = E, so a
deeper exit sees fewer perturbed layers (higher alpha), as in the paper.

    python tools/exit_sweep.py [--deep-scale 0.08] [--tokens 512] [--out profiles/r01_exit_sweep.json]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--deep-scale", type=float, default=0.08)
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--exits", default="4,8,12,16")
    ap.add_argument("--gammas", default="5,10")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
    rng = ppsd.RngStream(ppsd.derive_seed(0, "run"))
    ps = rng.split("prompt")
    prompt = [ps.randbelow(config.vocab) for _ in range(128)]
    rows = []
    for E in [int(x) for x in args.exits.split(",")]:
        lm = ppsd.TransformerLM(config, seed=0, deep_scale=args.deep_scale, deep_from=E)
        cfg = ppsd.PipelineConfig(config.n_layers, E)
        eng = ppsd.engine_for(lm, cfg)
        eng.set_schedule("pipelined")
        eng.decode(prompt, 64)  # warm-up (graphs, caches)
        tp, mp, trp = eng.decode(prompt, args.tokens)
        pipe_ms = eng.last["decode_ms"]
        eng.set_schedule("auto")
        eng.decode(prompt, 64)
        toks, m, tr = eng.decode(prompt, args.tokens)
        ppsd_ms = eng.last["decode_ms"]
        sched = eng.last["schedule"]
        assert tp == toks and mp == m and trp.to_csv() == tr.to_csv(), "schedules must agree"
        ar = eng.decode_ar(prompt, args.tokens)
        ar_ms = eng.last["decode_ms"]
        assert ar == toks, "PPSD must equal AR"
        row = dict(E=E, n_stages=cfg.n_stages, alpha_ppsd=m.alpha_all_measured, ticks=m.ticks,
                   schedule=sched, ppsd_tok_s=args.tokens / ppsd_ms * 1e3,
                   ppsd_pipelined_tok_s=args.tokens / pipe_ms * 1e3, ar_tok_s=args.tokens / ar_ms * 1e3,
                   ppsd_vs_ar=ar_ms / ppsd_ms, tick_speedup=m.speedup_vs_ar,
                   eq7=ppsd.ppsd_speedup(m.alpha_all_measured, config.n_layers, E))
        for g in [int(x) for x in args.gammas.split(",")]:
            et, em, _ = eng.decode_eesd(prompt, args.tokens, g)
            ems = eng.last["decode_ms"]
            assert et[: args.tokens] == toks, "EESD must equal AR"
            a = em.alpha_all_measured
            row[f"eesd_g{g}"] = dict(
                alpha_all=a, tok_s=em.committed_tokens / ems * 1e3, vs_ar=(em.committed_tokens / ems) / (args.tokens / ar_ms),
                tick_speedup=em.speedup_vs_ar)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del eng, lm
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(dict(deep_scale=args.deep_scale, tokens=args.tokens, prompt_len=128, rows=rows), fh, indent=1)


if __name__ == "__main__":
    main()
