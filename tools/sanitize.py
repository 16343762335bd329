"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the tiny transformer (PPSD folded + pipelined, AR, EESD) and a
2-layer Llama-2-7B-shaped model (PPSD folded, AR, EESD; tcgen05 GEMVs with
4-CTA split-K clusters for O / down, batched prefill), greedy.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "tiny"):
        lm = ppsd.TransformerLM(ppsd.TransformerConfig.tiny(8), seed=1, deep_scale=0.2, deep_from=2)
        cfg = ppsd.PipelineConfig(8, 2)
        prompt = [int(t) for t in np.random.default_rng(0).integers(0, 256, size=70)]
        ar = ppsd.decode_autoregressive(lm, prompt, 24, "greedy", ppsd.RngStream(0))
        for sched in ("folded", "pipelined"):
            lm.schedule = sched
            toks, m, _ = ppsd.decode_ppsd(lm, cfg, prompt, 24, "greedy", ppsd.RngStream(0))
            assert toks == ar, sched
        et, _, _ = ppsd.decode_eesd(lm, cfg, prompt, 24, 3)
        assert et[:24] == ar
        print("tiny ok", m.accepts, m.rejects)
    if which in ("all", "7b"):
        config = ppsd.TransformerConfig(2, 4096, 32, 32, 128, 11008, 32000, kv_dtype="bf16", max_ctx=256)
        lm = ppsd.TransformerLM(config, seed=2, deep_scale=0.3, deep_from=1)
        cfg = ppsd.PipelineConfig(2, 1)
        prompt = [int(t) for t in np.random.default_rng(1).integers(0, 32000, size=70)]
        ar = ppsd.decode_autoregressive(lm, prompt, 8, "greedy", ppsd.RngStream(0))
        toks, m, _ = ppsd.decode_ppsd(lm, cfg, prompt, 8, "greedy", ppsd.RngStream(0))
        assert toks == ar
        et, _, _ = ppsd.decode_eesd(lm, cfg, prompt, 8, 3)
        assert et[:8] == ar
        print("7b-2layer ok", m.accepts, m.rejects)


if __name__ == "__main__":
    main()
