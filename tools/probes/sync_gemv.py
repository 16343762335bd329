"""One GEMV probe launch of a 4-layer 7B-shaped engine, for compute-sanitizer
bisection: PPSD_TC_EXP bits (1 = no weight copies, 2 = no operand stores) are
applied through the trace switch.

    compute-sanitizer --tool synccheck python tools/probes/sync_gemv.py {qkv|o|gate_up|down} [groups]
"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200 import _lib  # noqa: E402
from paper_2509_19368_b200.decode import Engine  # noqa: E402

names = ["qkv", "o", "gate_up", "down", "head", "headv"]
which = names.index(sys.argv[1] if len(sys.argv) > 1 else "qkv")
groups = int(sys.argv[2]) if len(sys.argv) > 2 else 1
config = dataclasses.replace(ppsd.TransformerConfig.llama2_7b(max_ctx=256), n_layers=4)
lm = ppsd.TransformerLM(config, seed=0)
eng = Engine(lm.model_desc(), lm.weights_struct(), ppsd.PipelineConfig(4, 1), device=lm.device.index)
_lib.check(_lib.lib().ppsd_debug_tc_trace(0, None), "exp")  # loads PPSD_TC_EXP
ms, b = eng.probe_gemv(which, groups, 1)
print(f"{names[which]} groups={groups}: ok {ms * 1e3:.1f} us")
