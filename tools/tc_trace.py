"""Pipeline timeline of CTA 0 of one tensor-core GEMV launch (7B shape).

    python tools/tc_trace.py {qkv|o|gate_up|down|head} [vectors]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200 import _lib  # noqa: E402

names = ["qkv", "o", "gate_up", "down", "head", "headv"]
which = names.index(sys.argv[1] if len(sys.argv) > 1 else "down")
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 1
config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
lm = ppsd.TransformerLM(config, seed=0, deep_scale=0.16, deep_from=8)
eng = ppsd.engine_for(lm, ppsd.PipelineConfig(32, 8))
L = _lib.lib()
eng.probe_gemv(which, 1 if nv == 1 else -nv, 5)
_lib.check(L.ppsd_debug_tc_trace(1, None), "trace")
eng.probe_gemv(which, 1 if nv == 1 else -nv, 1)
buf = (C.c_uint64 * (8 * 128 + 160 * 4))()
_lib.check(L.ppsd_debug_tc_trace(0, buf), "trace")
allt = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
t = allt[:1024].reshape(8, 128)
cta = allt[1024:].reshape(160, 4)
t0 = t[6, 0]
rel = lambda x: (x - t0) / 1000.0 if x > 0 else float("nan")  # noqa: E731
print(f"{names[which]} nv={nv}: us after kernel start; cols: produced, mma_saw_full, mma_issued, built")
for n in range(128):
    if t[0, n] == 0 and t[1, n] == 0:
        break
    print(f"stage {n:3d}: {rel(t[0, n]):7.2f} {rel(t[1, n]):7.2f} {rel(t[2, n]):7.2f} {rel(t[3, n]):7.2f}")
print("startup: work read %.2f, barriers %.2f, syncthreads %.2f, cluster %.2f, weight ptr %.2f" %
      tuple(rel(t[7, i]) for i in range(5)))
print("producer: entry %.2f, policy %.2f, first tile %.2f, expect_tx %.2f, first copy issued %.2f" %
      tuple(rel(t[7, i]) for i in range(5, 10)))
for i in range(4):
    if t[4, i] > 0:
        print(f"tile {i}: epilogue saw acc_full at {rel(t[4, i]):7.2f}")

live = cta[cta[:, 0] > 0]
base = live[:, 0].min()
for k, name in enumerate(["start", "first copy", "last MMA issued", "exit"]):
    v = (live[:, k] - base) / 1000.0
    print(f"{name:16s} min {v.min():7.2f} p50 {np.median(v):7.2f} max {v.max():7.2f}  (us from the first CTA start)")
