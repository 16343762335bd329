"""AR decode timing of the 7B-shaped engine (CUDA events), for A/B experiments
such as PPSD_PROFILE_SKIP_ATTN=1 (attention's live share; wrong tokens).

    python tools/ar_profile.py [tokens]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=0.08, deep_from=8)
    ps = ppsd.RngStream(ppsd.derive_seed(0, "run")).split("prompt")
    prompt = [ps.randbelow(config.vocab) for _ in range(128)]
    eng = ppsd.engine_for(lm, ppsd.PipelineConfig(32, 8))
    eng.decode_ar(prompt, 16)
    best = None
    for _ in range(3):
        eng.decode_ar(prompt, n)
        ms = eng.last["decode_ms"]
        best = ms if best is None else min(best, ms)
    print(f"AR {n} tokens: {best:.2f} ms = {best / n * 1e3:.1f} us/token, {n / best * 1e3:.1f} tok/s "
          f"(skip_attn={os.environ.get('PPSD_PROFILE_SKIP_ATTN', '0')})", flush=True)


if __name__ == "__main__":
    main()
