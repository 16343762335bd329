"""CPU-side checks of the product boundary (no GPU needed)."""

import ctypes as C
import re
import os

import pytest

from conftest import ROOT


def test_library_loads_and_exports_every_header_symbol():
    from paper_2509_19368_b200 import _lib

    L = _lib.load_library()
    header = open(os.path.join(ROOT, "include", "ppsd.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(ppsd_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    for name in declared:
        assert getattr(L, name) is not None
    assert b"sm_100a" in L.ppsd_build_info()


def test_struct_layouts_match_header():
    from paper_2509_19368_b200 import _lib

    # sizes follow the C declarations (natural alignment, LP64)
    assert C.sizeof(_lib.ModelDesc) == 4 * 12 + 8 + 8 + 8
    assert C.sizeof(_lib.PipelineDesc) == 8 * 4
    assert C.sizeof(_lib.TraceRowC) == 24
    assert C.sizeof(_lib.Metrics) == 4 * 8 + 8 + 5 * 8 + 8 + 8 + 4 * 8
    # ...and what gcc computes from include/ppsd.h itself
    import subprocess
    import tempfile

    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "ppsd.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(ppsd_model_desc), sizeof(ppsd_pipeline_desc),
         sizeof(ppsd_metrics), sizeof(ppsd_trace_row), offsetof(ppsd_metrics, schedule),
         offsetof(ppsd_metrics, deep_pos_sum), sizeof(ppsd_weights), offsetof(ppsd_weights, exit_layer),
         offsetof(ppsd_metrics, comb_heads));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        with open(os.path.join(d, "s.c"), "w") as fh:
            fh.write(src)
        exe = os.path.join(d, "s")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, os.path.join(d, "s.c")])
        got = [int(x) for x in subprocess.check_output([exe], text=True).split()]
    assert got == [C.sizeof(_lib.ModelDesc), C.sizeof(_lib.PipelineDesc), C.sizeof(_lib.Metrics),
                   C.sizeof(_lib.TraceRowC), _lib.Metrics.schedule.offset, _lib.Metrics.deep_pos_sum.offset,
                   C.sizeof(_lib.Weights), _lib.Weights.exit_layer.offset, _lib.Metrics.comb_heads.offset]


def test_sm100a_cubin_embedded():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", os.path.join(ROOT, "paper_2509_19368_b200", "libppsd.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_engine_refuses_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2509_19368_b200 as ppsd

    with pytest.raises(RuntimeError):
        ppsd.decode_ppsd(ppsd.ToyLM(32, 16, 1, 1.0), ppsd.PipelineConfig(32, 8), [1], 4, "greedy",
                         ppsd.RngStream(0))


def test_host_api_mirrors_reference():
    import paper_2509_19368_b200 as ppsd

    cfg = ppsd.PipelineConfig(33, 8)
    assert cfg.n_stages == 5 and cfg.stage_layers == (8, 8, 8, 8, 1) and cfg.exit_stage == 1
    assert ppsd.PipelineConfig(32, 32).exit_stage is None
    with pytest.raises(ValueError):
        ppsd.PipelineConfig(32, 8, exit_stage=4)
    with pytest.raises(ValueError):
        ppsd.PipelineConfig(32, 0)
    assert ppsd.default_prompt(16, ppsd.RngStream(ppsd.derive_seed(0, "run"))) == [2, 6, 7, 7, 14, 2, 13, 13]
    assert abs(ppsd.ppsd_speedup(0.3226, 32, 8) - 1.319) <= 0.005
    m = ppsd.simulate_autoregressive(ppsd.PipelineConfig(40, 16), 10)
    assert m.ticks == 30


def test_tc_tiled_layout_python_matches_library():
    """paper_2509_19368_b200.tc_tile (the host-side checkpoint tiler) places
    every element where the library's ppsd_tc_offset (csrc/kernels.cuh, the
    layout the tensor-core GEMV and the device initialiser use) says, the
    padding is zero, and the layout is a bijection onto rows x padded cols."""
    import numpy as np
    import paper_2509_19368_b200 as ppsd
    from paper_2509_19368_b200 import _lib

    L = _lib.load_library()
    rng = np.random.default_rng(0)
    for rows, cols in ((8, 64), (24, 176), (352, 64), (64, 1024), (16, 11008 // 8 * 8), (40, 13824)):
        w = rng.standard_normal((rows, cols)).astype(np.float32)
        t = ppsd.tc_tile(w)
        n = C.c_int64()
        assert L.ppsd_weight_elems(1, rows, cols, C.byref(n)) == 0 and n.value == t.size
        # bijection: every logical element lands on its own slot, the rest is padding
        idx = np.zeros(t.size, dtype=np.int64)
        off = C.c_int64()
        for r in rng.integers(0, rows, size=12):
            for k in rng.integers(0, cols, size=12):
                assert L.ppsd_tc_offset(rows, cols, int(r), int(k), C.byref(off)) == 0
                assert t[off.value] == w[r, k]
        js, kp = ppsd.models.tc_layout(rows, cols)
        for r in range(0, rows, max(1, rows // 8)):
            for k in range(0, kp, 8):
                assert L.ppsd_tc_offset(rows, cols, r, k, C.byref(off)) == 0
                idx[off.value] += 1
        assert idx.max() <= 1
        # the tiled array holds exactly the matrix's elements plus zero padding
        assert np.array_equal(np.sort(t[t != 0]), np.sort(w[w != 0].ravel()))
