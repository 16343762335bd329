"""Per-tick cost of the multi-rank exchange, measured on one GPU.

A world=1 StageShard owns every stage and exchanges its box with itself over
the peer-store transport (pack kernel, per-thread system-scope fences, one
release store of the flag, the acquire-wait in the scheduler kernel). The
same model decoded by the single-device engine in the pipelined schedule
runs the identical layer kernels without the exchange, so the per-tick
difference of decode_ms / ticks is the exchange's device-side cost (NVLink
latency between GPUs comes on top). Tokens must match.

    python tools/p2p_overhead.py [--model 7b] [--exit 8] [--tokens 128]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200.distributed import StageShard, decode_ppsd_p2p, p2p_connect, p2p_prepare  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b")
    ap.add_argument("--exit", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    config = bench.model_config(args.model)
    cfg = ppsd.PipelineConfig(config.n_layers, args.exit)
    prompt = bench.bench_prompt(config.vocab)
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=bench.DEEP_SCALE, deep_from=args.exit)
    lm.schedule = "pipelined"
    eng = ppsd.engine_for(lm, cfg)
    single = []
    for _ in range(args.reps + 1):
        toks, m, _ = eng.decode(prompt, args.tokens, trace=False)
        single.append(eng.last["decode_ms"] / m.ticks)
    del eng, lm
    import gc

    gc.collect()
    shard = StageShard(config, cfg, 0, 1, seed=0, deep_scale=bench.DEEP_SCALE, deep_from=args.exit)
    _, xb = p2p_prepare(shard)
    p2p_connect(shard, local_xbufs=[xb])
    p2p = []
    for _ in range(args.reps + 1):
        t2, m2, _ = decode_ppsd_p2p(shard, prompt, args.tokens)
        p2p.append(shard.last["decode_ms"] / shard.last["ticks"])
    s, p = statistics.median(single[1:]), statistics.median(p2p[1:])
    print(json.dumps({"model": args.model, "exit": args.exit, "tokens": args.tokens, "ticks": m.ticks,
                      "single_us_per_tick": round(s * 1e3, 2), "p2p_us_per_tick": round(p * 1e3, 2),
                      "exchange_us_per_tick": round((p - s) * 1e3, 2), "tokens_equal": t2 == toks}))


if __name__ == "__main__":
    main()
