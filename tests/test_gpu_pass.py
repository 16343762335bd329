"""The persistent layer pass (csrc/tcpass.cu, opt-in PPSD_PASS=1) is the
per-kernel sequence's arithmetic in one launch per tick: the same tokens,
metrics and trace for PPSD (folded schedule) and AR. The pass takes split-K
clusters of at most 2 CTAs, so both runs force PPSD_TC_CS=1 (same plans)."""
import os

import numpy as np
import pytest

ppsd = pytest.importorskip("paper_2509_19368_b200")

pytestmark = pytest.mark.gpu


def test_layer_pass_equals_kernel_sequence():
    from paper_2509_19368_b200.decode import Engine

    config = ppsd.TransformerConfig(4, 4096, 32, 32, 128, 11008, 32000, kv_dtype="bf16", max_ctx=256)
    lm = ppsd.TransformerLM(config, seed=4, deep_scale=0.3, deep_from=2)
    cfg = ppsd.PipelineConfig(4, 2)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, config.vocab, size=40)]
    runs = {}
    for mode in ("0", "1"):
        os.environ["PPSD_PASS"], os.environ["PPSD_TC_CS"] = mode, "1"
        try:
            eng = Engine(lm.model_desc(), lm.weights_struct(), cfg, device=lm.device.index)
        finally:
            os.environ.pop("PPSD_PASS", None)
            os.environ.pop("PPSD_TC_CS", None)
        toks, m, tr = eng.decode(prompt, 24)
        launches = eng.last["gpu_launches"]
        ar = eng.decode_ar(prompt, 24)
        runs[mode] = (toks, (m.ticks, m.accepts, m.rejects), tr.to_csv(), ar, launches)
        del eng
    assert runs["0"][:4] == runs["1"][:4]
    assert runs["1"][0] == runs["1"][3]
    assert runs["1"][4] < runs["0"][4]  # the pass engaged: fewer launches per tick
