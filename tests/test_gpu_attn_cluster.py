"""Cluster decode attention (csrc/attn.cu: attn_cl_kernel, one-vector
launches) against the split-K kernel (PPSD_ATTN_CL=0): same tokens, metrics
and trace, and PPSD == AR, at contexts of one to more than kMergePages (32)
pages per row, which covers pages per rank > 1 and the global-partials path."""
import os

import numpy as np
import pytest

ppsd = pytest.importorskip("paper_2509_19368_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_prompt", [40, 700, 2100])
def test_cluster_attention_equals_split_k(n_prompt):
    from paper_2509_19368_b200.decode import Engine

    config = ppsd.TransformerConfig(4, 512, 4, 4, 128, 1408, 2048, kv_dtype="bf16", max_ctx=2300)
    lm = ppsd.TransformerLM(config, seed=12, deep_scale=0.3, deep_from=2)
    cfg = ppsd.PipelineConfig(4, 2)
    prompt = [int(t) for t in np.random.default_rng(n_prompt).integers(0, config.vocab, size=n_prompt)]
    runs = {}
    for mode in ("0", "1"):
        os.environ["PPSD_ATTN_CL"] = mode
        try:
            eng = Engine(lm.model_desc(), lm.weights_struct(), cfg, device=lm.device.index)
        finally:
            os.environ.pop("PPSD_ATTN_CL", None)
        toks, m, tr = eng.decode(prompt, 40)
        ar = eng.decode_ar(prompt, 40)
        runs[mode] = (toks, (m.ticks, m.accepts, m.rejects), tr.to_csv(), ar)
        del eng
    assert runs["0"] == runs["1"]
    assert runs["1"][0] == runs["1"][3]


@pytest.mark.parametrize("n_prompt,n_layers,exit_depth", [(40, 4, 1), (700, 8, 2), (2100, 4, 1)])
def test_batched_cluster_attention_equals_split_k(n_prompt, n_layers, exit_depth):
    """Folded deep batches (several vectors per group) on clusters of 4
    (PPSD_ATTN_CLB default) against the split-K kernel (PPSD_ATTN_CLB=0):
    same tokens, metrics and trace, and PPSD == AR."""
    from paper_2509_19368_b200.decode import Engine

    config = ppsd.TransformerConfig(n_layers, 512, 4, 4, 128, 1408, 2048, kv_dtype="bf16", max_ctx=2300)
    lm = ppsd.TransformerLM(config, seed=5, deep_scale=0.3, deep_from=exit_depth)
    cfg = ppsd.PipelineConfig(n_layers, exit_depth)
    prompt = [int(t) for t in np.random.default_rng(n_prompt).integers(0, config.vocab, size=n_prompt)]
    runs = {}
    for mode in ("0", "1"):
        os.environ["PPSD_ATTN_CLB"] = mode
        try:
            eng = Engine(lm.model_desc(), lm.weights_struct(), cfg, device=lm.device.index)
        finally:
            os.environ.pop("PPSD_ATTN_CLB", None)
        eng.set_schedule("folded")
        toks, m, tr = eng.decode(prompt, 48)
        ar = eng.decode_ar(prompt, 48)
        runs[mode] = (toks, (m.ticks, m.accepts, m.rejects), tr.to_csv(), ar)
        del eng
    assert runs["0"] == runs["1"]
    assert runs["1"][0] == runs["1"][3]
