"""Tiny transformer: pipelined-schedule PPSD vs AR tokens (sanitizer repro)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2509_19368_b200 as ppsd  # noqa: E402

lm = ppsd.TransformerLM(ppsd.TransformerConfig.tiny(8), seed=1, deep_scale=0.2, deep_from=2)
cfg = ppsd.PipelineConfig(8, 2)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, 256, size=70)]
ar = ppsd.decode_autoregressive(lm, prompt, 24, "greedy", ppsd.RngStream(0))
order = sys.argv[1:] or ["pipelined"]
for sched in order:
    lm.schedule = sched
    toks, m, _ = ppsd.decode_ppsd(lm, cfg, prompt, 24, "greedy", ppsd.RngStream(0))
    print(sched, "equal" if toks == ar else "DIFF", m.accepts, m.rejects)
    if toks != ar:
        print(" ar  ", ar)
        print(" ppsd", toks)
