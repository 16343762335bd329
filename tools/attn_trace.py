"""Timeline of the decode-attention workers' first items (7B shape, probe
launches): per event, the median / max over workers in us after the earliest
worker start. Needs libppsd built with EXTRA_NVFLAGS=-DPPSD_ATTN_TRACE.

    python tools/attn_trace.py [n_vec] [ctx]
"""
import ctypes as C
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200 import _lib  # noqa: E402
from paper_2509_19368_b200.decode import Engine  # noqa: E402

EV = ["start", "desc", "inputs", "q", "kv", "scores", "softmax", "partial", "ticket", "merged", "done"]


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 640
    config = dataclasses.replace(ppsd.TransformerConfig.llama2_7b(max_ctx=1024), n_layers=4)
    lm = ppsd.TransformerLM(config, seed=0)
    eng = Engine(lm.model_desc(), lm.weights_struct(), ppsd.PipelineConfig(4, 1), device=lm.device.index)
    L = _lib.lib()
    ms, _ = eng.probe_attn(nv, ctx, 50)
    _lib.check(L.ppsd_debug_tc_trace(5, None), "trace")
    eng.probe_attn(nv, ctx, 1)
    _lib.check(L.ppsd_debug_tc_trace(4, None), "trace")
    buf = (C.c_uint64 * (1024 * 12))()
    _lib.check(L.ppsd_debug_tc_trace(-4, buf), "trace")
    t = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(1024, 12)
    act = t[:, 4] > 0  # workers that had an item
    t0 = t[act, 0].min()
    print(f"n_vec={nv} ctx={ctx}: {ms * 1e3:.2f} us per launch back to back; {act.sum()} workers with items")
    for k, name in enumerate(EV):
        col = t[act, k]
        col = col[col > 0]
        if len(col) == 0:
            continue
        r = (col - t0) / 1e3
        print(f"{name:8s} n={len(col):4d}  min {r.min():6.2f}  med {np.median(r):6.2f}  max {r.max():6.2f}")
    # the last item's (merged) end relative to start: critical path
    eng.close()


if __name__ == "__main__":
    main()
