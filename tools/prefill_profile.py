"""Prompt prefill of the 7B-shaped engine (128 tokens), for a launch list:

    ncu --metrics gpu__time_duration.sum --csv python tools/prefill_profile.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=0.08, deep_from=8)
    ps = ppsd.RngStream(ppsd.derive_seed(0, "run")).split("prompt")
    prompt = [ps.randbelow(config.vocab) for _ in range(128)]
    toks, m, _ = ppsd.decode_ppsd(lm, ppsd.PipelineConfig(32, 8), prompt, 1, "greedy", ppsd.RngStream(0))
    print("prefill_ms", ppsd.engine_for(lm, ppsd.PipelineConfig(32, 8)).last.get("prefill_ms"))


if __name__ == "__main__":
    main()
