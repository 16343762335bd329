"""Time each layer GEMV of the 7B-shaped engine with CUDA events (and run under ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2509_19368_b200 as ppsd

def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=0.16, deep_from=8)
    eng = ppsd.engine_for(lm, ppsd.PipelineConfig(32, 8))
    names = ["qkv", "o", "gate_up", "down", "head"]
    for which in range(5):
        for g in ((1, 4) if which != 4 else (1,)):
            ms, b = eng.probe_gemv(which, g, reps)
            print(f"{names[which]:8s} groups={g} {b/1e6:8.1f} MB  {ms*1e3:8.1f} us  {b/ms/1e6:8.1f} GB/s", flush=True)

if __name__ == "__main__":
    main()
