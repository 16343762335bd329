"""One short folded PPSD decode of the 7B-shaped model, for ncu launch lists.

    PPSD_FOLD_COND=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum \
        --clock-control none -s 2400 -c 1500 --csv --log-file out.csv \
        python tools/fold_profile.py [tokens] [schedule]

PPSD_FOLD_COND=0 captures the deep part of the folded tick inline (ncu does
not profile graphs with conditional nodes); ticks without a deep batch then
launch its kernels with no work (filter them with launch_table.py --min-us).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    sched = sys.argv[2] if len(sys.argv) > 2 else "auto"
    config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
    cfg = ppsd.PipelineConfig(config.n_layers, 8)
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=0.08, deep_from=8)
    lm.schedule = sched
    rng = ppsd.RngStream(ppsd.derive_seed(0, "run"))
    ps = rng.split("prompt")
    prompt = [ps.randbelow(config.vocab) for _ in range(128)]
    eng = ppsd.engine_for(lm, cfg)
    toks, m, _ = eng.decode(prompt, n)
    print(f"{eng.last['schedule']}: {n} tokens {eng.last['decode_ms']:.2f} ms, ticks {m.ticks}, "
          f"accepts {m.accepts}, launches {eng.last['gpu_launches']}", flush=True)


if __name__ == "__main__":
    main()
