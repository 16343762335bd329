"""Sampling mode on the GPU against the reference.

ToyLM: tokens, metrics and trace must equal the reference's sampling runs
(tests/golden/toylm_sampling.json) — the device reproduces the stream draws,
numpy's pairwise summation and the inverse-CDF fold; only exp() may differ
by an ulp, which would move a sample only for a draw within ~1e-16 of a CDF
boundary. Transformer: lossless in distribution (first-token law)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
ppsd = pytest.importorskip("paper_2509_19368_b200")

CASES = load_golden("toylm_sampling.json")


def _ml(m):
    return [m.committed_tokens, m.ticks, m.accepts, m.rejects, m.alpha_all_measured, m.throughput,
            m.speedup_vs_ar]


@pytest.mark.parametrize("case", [c for c in CASES if c.get("kind") != "simulate"], ids=lambda c: c["name"])
def test_toylm_sampling_matches_reference(case):
    lm = ppsd.ToyLM(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    d = case["cfg"]
    cfg = ppsd.PipelineConfig(d["n_layers"], d["exit_depth"], exit_stage=d.get("exit_stage"),
                              comm_latency=d.get("comm_latency", 0))
    rng = ppsd.RngStream(case["rng_seed"])
    toks, m, tr = ppsd.decode_ppsd(lm, cfg, case["prompt"], case["max_tokens"], "sampling", rng)
    assert toks == case["tokens"]
    assert _ml(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]
    assert ppsd.decode_autoregressive(lm, case["prompt"], case["max_tokens"], "sampling", rng) == case["ar_tokens"]
    _, mf, _ = ppsd.decode_ppsd(lm, cfg, case["prompt"], case["max_tokens"], "sampling", rng, force_reject=True)
    assert _ml(mf) == case["force_reject_metrics"]


@pytest.mark.parametrize("case", [c for c in CASES if c.get("kind") == "simulate"], ids=lambda c: c["name"])
def test_simulate_ppsd_toy_sampling_matches_reference(case):
    lm = ppsd.ToyLM(32, 16, case["lm_seed"], case["beta"])
    tr = ppsd.EventTrace()
    m = ppsd.simulate_ppsd(ppsd.PipelineConfig(32, 8), ppsd.AcceptanceOracle.toylm_sampling(lm),
                           case["max_tokens"], ppsd.RngStream(case["rng_seed"]), trace=tr)
    assert _ml(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]


def test_transformer_sampling_first_token_law():
    """Lossless sampling: the first PPSD token is distributed as the target q
    (test_pipesim.py:405-415: V=16, 4000 seeds, TV < 0.05)."""
    config = ppsd.TransformerConfig(4, 256, 4, 4, 64, 704, 16, kv_dtype="fp32", max_ctx=128)
    lm = ppsd.TransformerLM(config, seed=2, deep_scale=1.0, deep_from=2)
    prompt = [3, 11, 7, 5]
    cfg = ppsd.PipelineConfig(4, 2)
    eng = ppsd.engine_for(lm, cfg)
    eng.decode_ar(prompt, 1)
    z = eng.read_logits(1).astype(np.float64)
    q = np.exp(z - z.max())
    q /= q.sum()
    n = 4000
    counts = np.zeros(config.vocab)
    for i in range(n):
        toks, _, _ = ppsd.decode_ppsd(lm, cfg, prompt, 1, "sampling", ppsd.RngStream(ppsd.derive_seed(i, "run")))
        counts[toks[0]] += 1
    tv = 0.5 * np.abs(counts / n - q).sum()
    assert tv < 0.05, tv


def test_transformer_sampling_force_reject_equals_ar():
    config = ppsd.TransformerConfig(6, 256, 4, 4, 64, 704, 512, kv_dtype="bf16", max_ctx=256)
    lm = ppsd.TransformerLM(config, seed=4, deep_scale=0.5, deep_from=2)
    prompt = [1, 2, 3, 4, 5]
    rng = ppsd.RngStream(77)
    toks, m, _ = ppsd.decode_ppsd(lm, ppsd.PipelineConfig(6, 2), prompt, 40, "sampling", rng, force_reject=True)
    assert toks == ppsd.decode_autoregressive(lm, prompt, 40, "sampling", rng)
    assert m.accepts == 0


def test_transformer_sampling_folded_equals_pipelined():
    """Sampling mode under the folded schedule (exit_stage 1: the eager exit
    logits are those of the draft tick; the batch's final logits are kept per
    vector) draws exactly what the pipelined schedule draws; exit_stage > 1
    sampling runs pipelined."""
    config = ppsd.TransformerConfig(8, 256, 4, 4, 64, 704, 512, kv_dtype="bf16", max_ctx=256)
    lm = ppsd.TransformerLM(config, seed=6, deep_scale=0.6, deep_from=2)
    prompt = [9, 8, 7, 6, 5, 4]
    cfg = ppsd.PipelineConfig(8, 2)
    out = {}
    for sched in ("pipelined", "folded"):
        lm.schedule = sched
        toks, m, tr = ppsd.decode_ppsd(lm, cfg, prompt, 60, "sampling", ppsd.RngStream(123))
        assert ppsd.engine_for(lm, cfg).schedule("sampling") == sched
        out[sched] = (toks, _ml(m), tr.to_csv())
    lm.schedule = "auto"
    assert out["folded"] == out["pipelined"]
    assert 0 < out["folded"][1][2] < 60  # both verdict kinds occur
    assert ppsd.engine_for(lm, ppsd.PipelineConfig(8, 2, exit_stage=2)).schedule("sampling") == "pipelined"


@pytest.mark.parametrize("case", load_golden("eesd_sampling.json"),
                         ids=lambda c: f"g{c['gamma']}-s{c['cfg'].get('exit_stage', 1)}")
def test_eesd_toy_sampling_matches_reference(case):
    """simulate_eesd with a toy sampling oracle (pipesim.py:435-551 with
    _ToyVerifier): drafts sampled from p, accept_draft / residual resample /
    bonus from the verify and commit streams — metrics and trace bit-exact."""
    lm = ppsd.ToyLM(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    tr = ppsd.EventTrace()
    m = ppsd.simulate_eesd(ppsd.PipelineConfig(**case["cfg"]), case["gamma"], ppsd.AcceptanceOracle.toylm_sampling(lm),
                           case["horizon"], ppsd.RngStream(case["rng_seed"]), trace=tr)
    assert _ml(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]


def test_transformer_eesd_sampling_first_token_law():
    """Lossless sampling EESD on the transformer: the first committed token
    follows the target q (accepted draft or residual resample)."""
    config = ppsd.TransformerConfig(4, 256, 4, 4, 64, 704, 16, kv_dtype="fp32", max_ctx=128)
    lm = ppsd.TransformerLM(config, seed=2, deep_scale=1.0, deep_from=2)
    prompt = [3, 11, 7, 5]
    cfg = ppsd.PipelineConfig(4, 2)
    eng = ppsd.engine_for(lm, cfg)
    eng.decode_ar(prompt, 1)
    z = eng.read_logits(1).astype(np.float64)
    q = np.exp(z - z.max())
    q /= q.sum()
    n = 3000
    counts = np.zeros(config.vocab)
    for i in range(n):
        toks, _, _ = ppsd.decode_eesd(lm, cfg, prompt, 1, 3, mode="sampling",
                                      rng=ppsd.RngStream(ppsd.derive_seed(i, "run")))
        counts[toks[0]] += 1
    tv = 0.5 * np.abs(counts / n - q).sum()
    assert tv < 0.06, tv
    a = ppsd.decode_eesd(lm, cfg, prompt, 30, 4, mode="sampling", rng=ppsd.RngStream(9))
    b = ppsd.decode_eesd(lm, cfg, prompt, 30, 4, mode="sampling", rng=ppsd.RngStream(9))
    assert a[0] == b[0] and a[2].to_csv() == b[2].to_csv()
