"""Where the end-to-end decode time goes beyond the device-timed decode and
prefill: wall clock of the public decode_ppsd call (bench workload) against
the engine's decode_ms + prefill_ms, and the wall clock of the bare C call.

    python tools/e2e_overhead.py [reps]
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200 import _lib  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    config = bench.model_config("7b")
    cfg = ppsd.PipelineConfig(config.n_layers, bench.EXIT_DEPTH)
    lm = ppsd.TransformerLM(config, seed=bench.SEED, deep_scale=bench.DEEP_SCALE, deep_from=bench.EXIT_DEPTH)
    prompt = bench.bench_prompt(config.vocab)
    eng = ppsd.engine_for(lm, cfg)
    ppsd.decode_ppsd(lm, cfg, prompt, bench.NEW_TOKENS, "greedy", ppsd.RngStream(0))
    rows = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ppsd.decode_ppsd(lm, cfg, prompt, bench.NEW_TOKENS, "greedy", ppsd.RngStream(0))
        wall = (time.perf_counter() - t0) * 1e3
        last = dict(eng.last)
        # the bare C call with the same buffers
        L = _lib.lib()
        p = (C.c_int32 * len(prompt))(*prompt)
        out = np.zeros(bench.NEW_TOKENS, dtype=np.int32)
        m = _lib.Metrics()
        cap = eng._trace_cap(bench.NEW_TOKENS)
        tr = np.zeros((cap, 6), dtype=np.int32)
        n = C.c_int64(0)
        t0 = time.perf_counter()
        _lib.check(L.ppsd_decode(eng.h, 1, 0, p, len(prompt), bench.NEW_TOKENS, 0,
                                 out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(m),
                                 tr.ctypes.data_as(C.POINTER(_lib.TraceRowC)), cap, C.byref(n)), "decode")
        c_wall = (time.perf_counter() - t0) * 1e3
        rows.append(dict(wall_ms=round(wall, 2), c_call_ms=round(c_wall, 2),
                         decode_ms=round(last["decode_ms"], 2), prefill_ms=round(last["prefill_ms"], 2),
                         c_decode_ms=round(m.decode_ms, 2), c_prefill_ms=round(m.prefill_ms, 2),
                         host_overhead_ms=round(wall - last["decode_ms"] - last["prefill_ms"], 2),
                         c_overhead_ms=round(c_wall - m.decode_ms - m.prefill_ms, 2)))
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
