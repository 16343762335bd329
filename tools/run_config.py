"""Run one BASELINE-shaped configuration on ONE GPU: PPSD vs AR (and EESD),
tokens/s, measured alpha, tick speedup, Eq. 7, step-level HBM roofline.

    python tools/run_config.py --model 13b --exit 20 --deep-scale 0.1
    python tools/run_config.py --model 70b --exit 10 --deep-scale 0.1 --tokens 256

On one GPU every stage shares one HBM; the same engine split
over S GPUs (paper_2509_19368_b200.distributed) realises the tick speedup.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=["7b", "13b", "70b"], default="7b")
    ap.add_argument("--exit", type=int, default=8)
    ap.add_argument("--deep-scale", type=float, default=0.08)
    ap.add_argument("--tokens", type=int, default=512)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--gamma", type=int, default=0, help="also run EESD with this gamma")
    ap.add_argument("--out", default=None)
    ap.add_argument("--schedule", default="auto", choices=["auto", "pipelined", "folded"])
    ap.add_argument("--exit-head", default="norm", choices=["norm", "layer"])
    args = ap.parse_args()
    config = {"7b": ppsd.TransformerConfig.llama2_7b, "13b": ppsd.TransformerConfig.llama2_13b,
              "70b": ppsd.TransformerConfig.llama2_70b}[args.model](max_ctx=args.prompt + args.tokens + 64)
    t0 = time.time()
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=args.deep_scale, deep_from=args.exit, exit_head=args.exit_head)
    init_s = time.time() - t0
    cfg = ppsd.PipelineConfig(config.n_layers, args.exit)
    rng = ppsd.RngStream(ppsd.derive_seed(0, "run"))
    ps = rng.split("prompt")
    prompt = [ps.randbelow(config.vocab) for _ in range(args.prompt)]
    eng = ppsd.engine_for(lm, cfg)
    eng.set_schedule("pipelined")
    eng.decode(prompt, 32)  # warm-up
    tp, mp, trp = eng.decode(prompt, args.tokens)
    pipe = dict(eng.last)
    eng.set_schedule(args.schedule)
    eng.decode(prompt, 32)
    toks, m, tr = eng.decode(prompt, args.tokens)
    pp = dict(eng.last)
    assert tp == toks and mp == m and trp.to_csv() == tr.to_csv(), "schedules must agree"
    ar = eng.decode_ar(prompt, args.tokens)
    ar_ms = eng.last["decode_ms"]
    assert ar == toks, "PPSD must equal AR"
    tr = trp  # the pipelined schedule's byte accounting (folded: see bench.py)
    fwd = sum(1 for r in tr if r.kind in ("ACTIVATION", "FINAL_TOKEN", "CHECK_TOKEN"))
    heads = len({r.tick for r in tr if r.kind in ("DRAFT_TOKEN", "FINAL_TOKEN", "CHECK_TOKEN")})
    kvb = config.kv_bytes_per_token_layer()
    kv = sum(cfg.stage_layers[r.stage - 1] * (args.prompt + r.position - 1) * kvb
             for r in tr if r.kind in ("ACTIVATION", "FINAL_TOKEN", "CHECK_TOKEN"))
    step_bytes = sum(cfg.stage_layers[r.stage - 1] for r in tr
                     if r.kind in ("ACTIVATION", "FINAL_TOKEN", "CHECK_TOKEN")) * config.layer_bytes() \
        + heads * config.head_bytes() + kv
    row = dict(model=config.name, exit_head=args.exit_head, weights_gb=round((config.n_layers * config.layer_bytes() + 2 * config.head_bytes()) / 1e9, 2),
               exit=args.exit, n_stages=cfg.n_stages, deep_scale=args.deep_scale, init_s=round(init_s, 1),
               alpha=m.alpha_all_measured, ticks=m.ticks, stage_forwards=fwd,
               schedule=pp["schedule"], ppsd_tok_s=round(args.tokens / pp["decode_ms"] * 1e3, 2),
               ppsd_pipelined_tok_s=round(args.tokens / pipe["decode_ms"] * 1e3, 2),
               deep_batches=pp["deep_batches"], deep_vectors=pp["deep_vectors"],
               ar_tok_s=round(args.tokens / ar_ms * 1e3, 2),
               ppsd_vs_ar=round(ar_ms / pp["decode_ms"], 4), tick_speedup=round(m.speedup_vs_ar, 4),
               eq7=round(ppsd.ppsd_speedup(m.alpha_all_measured, config.n_layers, args.exit), 4),
               pipelined_step_gbs=round(step_bytes / (pipe["decode_ms"] / 1e3) / 1e9, 1),
               prefill_ms=round(pp["prefill_ms"], 1))
    if args.gamma:
        et, em, _ = eng.decode_eesd(prompt, args.tokens, args.gamma)
        assert et[: args.tokens] == toks, "EESD must equal AR"
        row["eesd"] = dict(gamma=args.gamma, alpha_all=em.alpha_all_measured,
                           tok_s=round(em.committed_tokens / eng.last["decode_ms"] * 1e3, 2),
                           tick_speedup=round(em.speedup_vs_ar, 4))
    print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(row, fh, indent=1)


if __name__ == "__main__":
    main()
