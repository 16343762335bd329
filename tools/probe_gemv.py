"""Time each layer GEMV of the 7B-shaped engine with CUDA events (and run under ncu).

    python tools/probe_gemv.py [reps] [matrix] [groups,...]   (negative = batched vectors)

Rows: the decode-tick plan (M=1) over 1 and 4 groups, and the batched plan
with 1-4 vectors (folded deep batch). Launches walk the stage's layers so no
launch finds its weights in L2.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    only = sys.argv[2] if len(sys.argv) > 2 else None
    pick = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
    config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
    lm = ppsd.TransformerLM(config, seed=0, deep_scale=0.16, deep_from=8)
    eng = ppsd.engine_for(lm, ppsd.PipelineConfig(32, 8))
    names = ["qkv", "o", "gate_up", "down", "head", "headv"]
    for which in range(6):
        if only and names[which] != only:
            continue
        groups = (1, 4, -1, -2, -3, -4) if which < 4 else ((1,) if which == 4 else (-1, -2, -4))
        for g in (pick or groups):
            ms, b = eng.probe_gemv(which, g, reps)
            lab = f"groups={g}" if g > 0 else f"vectors={-g}"
            print(f"{names[which]:8s} {lab:10s} {b/1e6:8.1f} MB  {ms*1e3:8.1f} us  {b/ms/1e6:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
