"""Measured greedy acceptance rate vs deep_scale on the 7B-shaped model (bench calibration)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_19368_b200 as ppsd

config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
cfg = ppsd.PipelineConfig(32, 8)
rng = ppsd.RngStream(ppsd.derive_seed(0, "run"))
ps = rng.split("prompt")
prompt = [ps.randbelow(config.vocab) for _ in range(128)]
for ds in [float(x) for x in sys.argv[1:]]:
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=ds, deep_from=8)
    eng = ppsd.engine_for(lm, cfg)
    toks, m, tr = eng.decode(prompt, 512)
    ms = eng.last["decode_ms"]
    ar = eng.decode_ar(prompt, 512)
    print(f"deep_scale={ds:5.3f} alpha={m.alpha_all_measured:.3f} ticks={m.ticks} ppsd={512/ms*1e3:7.1f} tok/s "
          f"ar={512/eng.last['decode_ms']*1e3:7.1f} tok/s equal={toks == ar} eq7={ppsd.ppsd_speedup(m.alpha_all_measured, 32, 8):.3f}",
          flush=True)
    del eng, lm
    torch.cuda.empty_cache()
