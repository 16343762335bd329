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
    assert C.sizeof(_lib.ModelDesc) == 4 * 12 + 8 + 8
    assert C.sizeof(_lib.PipelineDesc) == 7 * 4
    assert C.sizeof(_lib.TraceRowC) == 24
    assert C.sizeof(_lib.Metrics) == 4 * 8 + 8 + 5 * 8 + 8


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
