"""Projected N-GPU PPSD throughput from per-rank stage times measured on ONE GPU.

The multi-rank engines of a world-W pipeline run as W engines on cuda:0
(loopback exchange, one rank at a time). Each rank's tick graph (its stages'
layers + heads + box pack) is timed with CUDA events on its own stream, and
so is the replicated scheduler step. On W GPUs the ranks run concurrently, so
a tick costs max over ranks (compute + scheduler) plus one box exchange.
The exchange is an input (--xfer-us, default 13.3 us: the device-side cost of
the peer-store exchange per tick measured on one GPU by tools/p2p_overhead.py;
the NVLink latency between two GPUs comes on top). Output is a projection, not
a bench number:

    python tools/project_multigpu.py --model 13b --exit 20 --world 2
    python tools/project_multigpu.py --model 70b --exit 10 --world 4 --tokens 128
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200.distributed import StageShard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=["7b", "13b", "70b"], default="13b")
    ap.add_argument("--exit", type=int, default=20)
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--deep-scale", type=float, default=0.1)
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--xfer-us", type=float, default=13.3)  # tools/p2p_overhead.py: loopback peer-store exchange, 7B
    ap.add_argument("--schedule", choices=["auto", "pipelined"], default="auto")  # auto: ranks fold where they can
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    presets = {"7b": ppsd.TransformerConfig.llama2_7b, "13b": ppsd.TransformerConfig.llama2_13b,
               "70b": ppsd.TransformerConfig.llama2_70b}
    config = presets[args.model](max_ctx=args.prompt + args.tokens + 64)
    cfg = ppsd.PipelineConfig(config.n_layers, args.exit)
    shards = [StageShard(config, cfg, r, args.world, seed=0, deep_scale=args.deep_scale, deep_from=args.exit)
              for r in range(args.world)]
    for s in shards:
        s.engine.set_schedule(args.schedule)
    ps = ppsd.RngStream(ppsd.derive_seed(0, "run")).split("prompt")
    prompt = [ps.randbelow(config.vocab) for _ in range(args.prompt)]

    def exchange():
        torch.cuda.synchronize()
        boxes = torch.stack([s.outbox for s in shards])
        for s in shards:
            s.inbox.copy_(boxes)
        torch.cuda.synchronize()

    def run(timed):
        steps = [s.begin(prompt, args.tokens) for s in shards][0]
        for _ in range(steps):
            for s in shards:
                s.prefill_compute()
            exchange()
        per_tick = []
        committed = 0
        while True:
            for _ in range(max(1, args.tokens - committed)):
                t = []
                for s in shards:  # one rank at a time: each is timed alone on the GPU
                    st = s.torch_stream()
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                    ev[0].record(st)
                    s.compute()
                    ev[1].record(st)
                    torch.cuda.synchronize()
                    t.append((s, ev, st))
                exchange()
                for s, ev, st in t:
                    ev[2].record(st)
                    s.finish()
                    ev[3].record(st)
                    torch.cuda.synchronize()
                if timed:
                    per_tick.append([(ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])) for _, ev, _ in t])
            done, committed, _ = shards[0].poll()
            if done:
                break
        return per_tick, [s.end() for s in shards]

    run(False)  # warm-up (graph capture, lazy loading)
    ticks, results = run(True)
    toks, m, _ = results[0]
    arr = np.array(ticks)  # [tick][rank][compute_ms, finish_ms]
    # the tick loop launches ticks past the last commit; count the machine's ticks
    used = arr[: m.ticks]
    rank_ms = used[:, :, 0] + used[:, :, 1]
    tick_ms = rank_ms.max(axis=1) + args.xfer_us / 1000.0
    total_s = float(tick_ms.sum()) / 1000.0
    out = {
        "kind": "projection (per-rank stage times measured on one B200; exchange modelled)",
        "model": args.model, "exit": args.exit, "world": args.world, "n_stages": cfg.n_stages,
        "tokens": args.tokens, "prompt": args.prompt, "deep_scale": args.deep_scale,
        "alpha": m.alpha_all_measured, "ticks": m.ticks, "committed": m.committed_tokens,
        "rank_compute_ms_mean": [round(float(x), 4) for x in used[:, :, 0].mean(axis=0)],
        "rank_sched_ms_mean": [round(float(x), 4) for x in used[:, :, 1].mean(axis=0)],
        "rank_schedule": [s.last["schedule"] for s in shards],
        "rank_deep_batches": [s.last["deep_batches"] for s in shards],
        "xfer_us_assumed": args.xfer_us,
        "projected_tick_ms": round(float(tick_ms.mean()), 4),
        "projected_tokens_per_s": round(m.committed_tokens / total_s, 2),
    }
    print(json.dumps(out))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
