"""Timeline of CTA 0 in one layer pass (build with EXTRA_NVFLAGS=-DPPSD_TC_TRACE).

    python tools/pass_trace.py [n_layers]
Runs one AR step of a 7B-shaped model and prints, for the first layers of the
pass: weight stages produced / consumed by the MMA, grid-barrier completions
seen by the builders and epilogues, and this CTA's barrier arrivals.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200 import _lib  # noqa: E402

nl = int(sys.argv[1]) if len(sys.argv) > 1 else 2
config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024, n_layers=nl)
lm = ppsd.TransformerLM(config, seed=0)
eng = ppsd.Engine(lm.model_desc(), lm.weights_struct(), ppsd.PipelineConfig(config.n_layers, 1),
                  device=lm.device.index)
L = _lib.lib()
prompt = list(range(1, 65))
eng.decode_ar(prompt, 3)
_lib.check(L.ppsd_debug_tc_trace(3, None), "trace")
eng.decode_ar(prompt, 2)
buf = (C.c_uint64 * (8 * 128))()
_lib.check(L.ppsd_debug_tc_trace(-2, buf), "trace")
_lib.check(L.ppsd_debug_tc_trace(2, None), "trace")
t = np.frombuffer(buf, dtype=np.uint64).reshape(8, 128).astype(np.int64)
t0 = t[6, 0]
rel = lambda x: (x - t0) / 1000.0 if x > 0 else float("nan")  # noqa: E731
print("stages: n produced mma_saw_full")
for n in range(128):
    if t[0, n] == 0:
        break
    print(f"  {n:3d} {rel(t[0, n]):8.2f} {rel(t[1, n]):8.2f}")
print("barriers: k builders_saw epilogue_saw epilogue_arrival(k-th arrival)")
for k in range(40):
    if t[2, k] == 0 and t[3, k] == 0:
        continue
    print(f"  {k:3d} {rel(t[2, k]):8.2f} {rel(t[3, k]):8.2f} {rel(t[4, k]):8.2f}")
for i in range(8):
    if t[5, i]:
        print(f"attention layer {i} arrival {rel(t[5, i]):8.2f}")
