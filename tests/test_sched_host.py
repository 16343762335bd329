"""The shipped tick machine (csrc/sched.h, host build) against reference goldens."""

import pytest

from conftest import load_golden
from hostsched import run_bernoulli, run_toy
from oracle import specpipe_port as sp


@pytest.mark.parametrize("case", load_golden("toylm_decode.json"), ids=lambda c: c["name"])
def test_sched_toy_matches_reference(case):
    lm = sp.ToyLMPort(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    cfg = case["cfg"]
    toks, m, rows = run_toy(lm, cfg["n_layers"], cfg["exit_depth"], case["prompt"],
                            case["max_tokens"], exit_stage=cfg.get("exit_stage", 0) or 0,
                            comm_latency=cfg.get("comm_latency", 0))
    assert toks == case["tokens"]
    assert list(m[:4]) == case["metrics"][:4]
    assert m[4:] == tuple(case["metrics"][4:])
    assert sp.trace_csv(rows) == case["trace_csv"]


@pytest.mark.parametrize("case", load_golden("bernoulli.json"), ids=lambda c: f"a{c['alpha']}-{c['horizon']}")
def test_sched_bernoulli_matches_reference(case):
    cfg = case["cfg"]
    verify_seed = sp.Stream(case["rng_seed"]).split("verify").seed
    m, rows = run_bernoulli(cfg["n_layers"], cfg["exit_depth"], case["alpha"], case["horizon"],
                            verify_seed, exit_stage=cfg.get("exit_stage", 0) or 0,
                            comm_latency=cfg.get("comm_latency", 0))
    assert list(m) == case["metrics"]
    assert sp.trace_csv(rows) == case["trace_csv"]


@pytest.mark.parametrize("case", load_golden("toylm_decode.json"), ids=lambda c: c["name"])
def test_sched_folded_matches_reference(case):
    """The folded single-device schedule (sched.h: sched_fold_plan) with eager
    drafts and batched deep verdicts reproduces the reference machine exactly,
    and every batch is the consecutive fold rows 0..nb-1 the kernels read."""
    from hostsched import run_toy_folded

    lm = sp.ToyLMPort(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    cfg = case["cfg"]
    S = -(-cfg["n_layers"] // cfg["exit_depth"])
    if (S - 1) * (1 + cfg.get("comm_latency", 0)) + 1 > 16:
        pytest.skip("more chains in flight than one batch holds: the engine runs this pipelined")
    toks, m, rows, batches = run_toy_folded(lm, cfg["n_layers"], cfg["exit_depth"], case["prompt"],
                                            case["max_tokens"],
                                            exit_stage=cfg.get("exit_stage", 0) or 0,
                                            comm_latency=cfg.get("comm_latency", 0),
                                            force_reject=case.get("force_reject", False))
    assert toks == case["tokens"]
    assert list(m[:4]) == case["metrics"][:4]
    assert m[4:] == tuple(case["metrics"][4:])
    assert sp.trace_csv(rows) == case["trace_csv"]
    if case["max_tokens"] > 0:
        # one deep pass verifies several chains: fewer passes than verdicts
        assert sum(batches) >= m[0] and len(batches) <= m[0]


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("case", load_golden("toylm_decode.json"), ids=lambda c: c["name"])
def test_sched_rank_folded_matches_reference(case, world):
    """Multi-rank with the per-rank fold (sched.h: sched_rfold_plan): every
    rank whose deferred stages span >= 2 stages batches them; tokens, metrics
    and trace stay the reference's, every input exists when a rank uses it,
    and folding ranks stream their deferred weights fewer times than ticks."""
    from hostsched import run_toy_multirank_folded

    lm = sp.ToyLMPort(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    cfg = case["cfg"]
    S = -(-cfg["n_layers"] // cfg["exit_depth"])
    if world > S:
        pytest.skip("more ranks than stages")
    toks, m, rows, batches = run_toy_multirank_folded(
        lm, cfg["n_layers"], cfg["exit_depth"], case["prompt"], case["max_tokens"], world,
        exit_stage=cfg.get("exit_stage", 0) or 0, comm_latency=cfg.get("comm_latency", 0),
        force_reject=case.get("force_reject", False))
    assert toks == case["tokens"]
    assert list(m[:4]) == case["metrics"][:4]
    assert m[4:] == tuple(case["metrics"][4:])
    assert sp.trace_csv(rows) == case["trace_csv"]
    for r, b in batches.items():
        assert len(b) <= m[1], (r, len(b), m[1])
