"""Sampling mode: the oracle port against reference goldens.

Sampling draws come from three counter streams (draft / verify / commit,
pipesim.py:339-344); the port runs the same numpy float64 ops as the
reference, so tokens, accept counts and traces are reproduced exactly."""

import pytest

from conftest import load_golden
from oracle import specpipe_port as sp

CASES = load_golden("toylm_sampling.json")


@pytest.mark.parametrize("case", [c for c in CASES if c.get("kind") != "simulate"], ids=lambda c: c["name"])
def test_sampling_decode_matches_reference(case):
    lm = sp.ToyLMPort(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    cfg = case["cfg"]
    kw = dict(exit_stage=cfg.get("exit_stage"), comm_latency=cfg.get("comm_latency", 0), greedy=False,
              rng_seed=case["rng_seed"])
    toks, m, rows = sp.decode_ppsd(lm, cfg["n_layers"], cfg["exit_depth"], case["prompt"], case["max_tokens"], **kw)
    assert toks == case["tokens"]
    assert list(m) == case["metrics"]
    assert sp.trace_csv(rows) == case["trace_csv"]
    assert sp.decode_autoregressive(lm, case["prompt"], case["max_tokens"], greedy=False,
                                    rng_seed=case["rng_seed"]) == case["ar_tokens"]
    _, mf, _ = sp.decode_ppsd(lm, cfg["n_layers"], cfg["exit_depth"], case["prompt"], case["max_tokens"],
                              force_reject=True, **kw)
    assert list(mf) == case["force_reject_metrics"]


@pytest.mark.parametrize("case", [c for c in CASES if c.get("kind") == "simulate"], ids=lambda c: c["name"])
def test_sampling_simulate_matches_reference(case):
    lm = sp.ToyLMPort(32, 16, case["lm_seed"], case["beta"])
    prompt = sp.default_prompt(16, case["rng_seed"])
    _, m, rows = sp.decode_ppsd(lm, 32, 8, prompt, case["max_tokens"], greedy=False, rng_seed=case["rng_seed"])
    assert list(m) == case["metrics"]
    assert sp.trace_csv(rows) == case["trace_csv"]
