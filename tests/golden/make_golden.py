"""Regenerate the golden fixtures from the REAL reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference `specpipe` package from /root/reference (read-only,
present only in the build container) and records its outputs as JSON so the
oracle port and the GPU path can be checked against them anywhere, including
the GPU box where /root/reference does not exist. Nothing at test/bench time
reads /root/reference.

Fixture files:
  toylm_decode.json   decode_ppsd / decode_autoregressive (greedy) on ToyLM
  bernoulli.json      simulate_ppsd (traced machine + untraced fast path)
  acceptance200.json  the 200-case sweep of test_acceptance.py:133-154
  eesd_toy.json       simulate_eesd with the toy greedy oracle + Bernoulli
  eesd_sampling.json  simulate_eesd with the toy sampling oracle
  transformer.json    reference decode_ppsd driving oracle/transformer.py
  transformer_head.json  the same with a decoder-layer exit head (exit_head_at)
  cli_decode.json     `specpipe decode` transcripts (stdout, exit code)
  cli_harness.json    `specpipe analytic|run|sweep|trace` transcripts (stdout,
                      stderr, exit code)
  harness.json        harness.run results rows (+ analytic column), ToyLM
                      empirical_alpha / greedy_agreement, ConfigError messages,
                      analytic_report
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import specpipe as sp  # noqa: E402
from specpipe.pipesim import EventTrace  # noqa: E402


def trace_text(trace) -> str:
    buf = io.StringIO()
    trace.write_csv(buf)
    return buf.getvalue()


def metrics_list(m) -> list:
    return [m.committed_tokens, m.ticks, m.accepts, m.rejects,
            m.alpha_all_measured, m.throughput, m.speedup_vs_ar]


def run_rng(seed):
    return sp.RngStream(sp.derive_seed(seed, "run"))


TOY_CASES = [
    # name, n_layers, vocab, lm seed label, beta, cfg kwargs, prompt, max_tokens
    ("survey_b0", 32, 16, 0, 0.0, dict(n_layers=32, exit_depth=8), None, 128),
    ("survey_b1", 32, 16, 0, 1.0, dict(n_layers=32, exit_depth=8), None, 128),
    ("survey_b2", 32, 16, 0, 2.0, dict(n_layers=32, exit_depth=8), None, 128),
    ("decode_lm3", 32, 16, 3, 1.0, dict(n_layers=32, exit_depth=8), [1, 2, 3, 4], 96),
    ("deep_exit", 32, 16, 5, 1.0, dict(n_layers=32, exit_depth=8, exit_stage=2), [6, 6], 48),
    ("comm_lat2", 32, 16, 5, 1.0, dict(n_layers=32, exit_depth=8, comm_latency=2), [6, 6], 48),
    ("remainder33", 33, 16, 7, 1.5, dict(n_layers=33, exit_depth=8), [9, 0, 2], 80),
    ("two_stage", 40, 16, 8, 0.7, dict(n_layers=40, exit_depth=20), [4], 64),
    ("eight_stage", 80, 16, 9, 1.0, dict(n_layers=80, exit_depth=10), [3, 1, 4, 1, 5], 100),
    ("vocab1000", 32, 1000, 10, 0.3, dict(n_layers=32, exit_depth=8), [17, 999, 0, 512], 128),
    ("vocab32000", 32, 32000, 11, 0.2, dict(n_layers=32, exit_depth=8), [1, 31999], 40),
    ("deep_exit3_lat1", 48, 16, 12, 1.0, dict(n_layers=48, exit_depth=8, exit_stage=3, comm_latency=1), [2, 2, 2], 60),
    ("single_token", 32, 16, 13, 1.0, dict(n_layers=32, exit_depth=8), [5], 1),
    ("zero_tokens", 32, 16, 13, 1.0, dict(n_layers=32, exit_depth=8), [5], 0),
]


def make_toy():
    out = []
    for name, n, vocab, seed, beta, cfgkw, prompt, max_tokens in TOY_CASES:
        lm = sp.ToyLM(n_layers=n, vocab=vocab, seed=sp.derive_seed(seed, "lm"), misalignment=beta)
        cfg = sp.PipelineConfig(**cfgkw)
        rng = run_rng(seed)
        if prompt is None:
            prompt = sp.default_prompt(vocab, rng)
        toks, m, tr = sp.decode_ppsd(lm, cfg, prompt, max_tokens, "greedy", run_rng(seed))
        ar = sp.decode_autoregressive(lm, prompt, max_tokens, "greedy", run_rng(seed))
        fr_toks, fr_m, _ = sp.decode_ppsd(lm, cfg, prompt, max_tokens, "greedy", run_rng(seed),
                                          force_reject=True)
        assert toks == ar == fr_toks
        out.append(dict(
            name=name, n_layers=n, vocab=vocab, lm_seed=lm.seed, beta=beta, cfg=cfgkw,
            prompt=list(map(int, prompt)), max_tokens=max_tokens, rng_seed=run_rng(seed).seed,
            tokens=toks, metrics=metrics_list(m), trace_csv=trace_text(tr), ar_tokens=ar,
            force_reject_metrics=metrics_list(fr_m)))
    return out


BERN_CASES = [
    # alpha, cfg kwargs, horizon, seed
    (0.6, dict(n_layers=32, exit_depth=8), 300, 0),
    (1.0, dict(n_layers=32, exit_depth=8), 200, 0),
    (0.0, dict(n_layers=32, exit_depth=8), 50, 1),
    (0.5, dict(n_layers=32, exit_depth=8), 200, 5),
    (0.7, dict(n_layers=33, exit_depth=8), 300, 11),
    (0.6, dict(n_layers=32, exit_depth=8, exit_stage=2), 300, 12),
    (0.8, dict(n_layers=32, exit_depth=8, comm_latency=1), 300, 13),
    (0.4, dict(n_layers=80, exit_depth=10), 500, 14),
    (0.9, dict(n_layers=40, exit_depth=20), 400, 15),
]


def make_bernoulli():
    out = []
    for alpha, cfgkw, horizon, seed in BERN_CASES:
        cfg = sp.PipelineConfig(**cfgkw)
        tr = EventTrace()
        m = sp.simulate_ppsd(cfg, sp.AcceptanceOracle.bernoulli(alpha), horizon, run_rng(seed), trace=tr)
        fast = sp.simulate_ppsd(cfg, sp.AcceptanceOracle.bernoulli(alpha), horizon, run_rng(seed))
        assert fast == m
        out.append(dict(alpha=alpha, cfg=cfgkw, horizon=horizon, rng_seed=run_rng(seed).seed,
                        metrics=metrics_list(m), trace_csv=trace_text(tr)))
    return out


def tokens_digest(tokens) -> str:
    return hashlib.sha256(",".join(map(str, tokens)).encode()).hexdigest()


def make_acceptance200():
    """Mirror of test_acceptance.py:133-154 inputs, with outputs recorded."""
    gen = np.random.default_rng(2026)
    cfg = sp.PipelineConfig(32, 8)
    cases = []
    for i in range(200):
        seed = int(gen.integers(2**63))
        lm = sp.ToyLM(n_layers=32, vocab=16, seed=seed, misalignment=1.0)
        prompt = [int(t) for t in gen.integers(16, size=8)]
        toks, m, _ = sp.decode_ppsd(lm, cfg, prompt, 256, "greedy", run_rng(i))
        cases.append(dict(lm_seed=seed, prompt=prompt, tokens_sha256=tokens_digest(toks),
                          first8=toks[:8], metrics=metrics_list(m)))
    return cases


def make_eesd():
    out = []
    for gamma, beta, seed in ((5, 1.0, 0), (3, 0.0, 1), (10, 2.0, 2), (1, 1.0, 3)):
        lm = sp.ToyLM(n_layers=32, vocab=16, seed=sp.derive_seed(seed, "lm"), misalignment=beta)
        cfg = sp.PipelineConfig(32, 8)
        tr = EventTrace()
        m = sp.simulate_eesd(cfg, gamma, sp.AcceptanceOracle.toylm_greedy(lm), 128, run_rng(seed), trace=tr)
        out.append(dict(kind="toy", gamma=gamma, beta=beta, lm_seed=lm.seed, rng_seed=run_rng(seed).seed,
                        horizon=128, metrics=metrics_list(m), trace_csv=trace_text(tr)))
    for gamma, alpha, seed in ((4, 0.5, 4), (10, 0.3, 5)):
        cfg = sp.PipelineConfig(32, 8)
        tr = EventTrace()
        m = sp.simulate_eesd(cfg, gamma, sp.AcceptanceOracle.bernoulli(alpha), 200, run_rng(seed), trace=tr)
        out.append(dict(kind="bernoulli", gamma=gamma, alpha=alpha, rng_seed=run_rng(seed).seed,
                        horizon=200, metrics=metrics_list(m), trace_csv=trace_text(tr)))
    return out


def make_transformer():
    """Reference decode_ppsd / decode_autoregressive driving the CPU fp64
    transformer oracle through the reference's own 7-member model protocol."""
    from oracle.transformer import TransformerOracle, tiny_config

    out = []
    for name, deep_scale, cfgkw, n_tok, seed in (
        ("tiny_ds010", 0.10, dict(n_layers=32, exit_depth=8), 128, 0),
        ("tiny_ds025", 0.25, dict(n_layers=32, exit_depth=8), 128, 1),
        ("tiny_ds000", 0.0, dict(n_layers=32, exit_depth=8), 64, 2),
        ("tiny_deep_exit", 0.15, dict(n_layers=32, exit_depth=8, exit_stage=2), 64, 3),
    ):
        mc = tiny_config()
        lm = TransformerOracle(mc, seed=seed, deep_scale=deep_scale, deep_from=8, dtype=np.float64)
        cfg = sp.PipelineConfig(**cfgkw)
        prompt = sp.default_prompt(mc.vocab, run_rng(seed))
        toks, m, tr = sp.decode_ppsd(lm, cfg, prompt, n_tok, "greedy", run_rng(seed))
        ar = sp.decode_autoregressive(lm, prompt, n_tok, "greedy", run_rng(seed))
        assert toks == ar, name
        out.append(dict(name=name, model=mc.to_dict(), seed=seed, deep_scale=deep_scale, deep_from=8,
                        cfg=cfgkw, prompt=prompt, max_tokens=n_tok, tokens=toks,
                        metrics=metrics_list(m), trace_csv=trace_text(tr),
                        min_margins=lm.margin_report()))
        print(name, metrics_list(m), flush=True)
    return out


def make_transformer_head():
    """As make_transformer, with the exit head of the paper's main runs: one
    decoder layer on the exit-layer state, then the norm head."""
    from oracle.transformer import TransformerOracle, tiny_config

    out = []
    for name, deep_scale, cfgkw, n_tok, seed in (
        ("tiny_hl_ds010", 0.10, dict(n_layers=32, exit_depth=8), 96, 5),
        ("tiny_hl_ds030", 0.30, dict(n_layers=32, exit_depth=8), 96, 6),
        ("tiny_hl_deep_exit", 0.15, dict(n_layers=32, exit_depth=8, exit_stage=2), 64, 7),
        ("tiny_hl_comm_lat", 0.20, dict(n_layers=32, exit_depth=8, comm_latency=1), 64, 8),
    ):
        mc = tiny_config()
        cfg = sp.PipelineConfig(**cfgkw)
        lm = TransformerOracle(mc, seed=seed, deep_scale=deep_scale, deep_from=8, dtype=np.float64,
                               exit_head_at=cfg.exit_layer)
        prompt = sp.default_prompt(mc.vocab, run_rng(seed))
        toks, m, tr = sp.decode_ppsd(lm, cfg, prompt, n_tok, "greedy", run_rng(seed))
        ar = sp.decode_autoregressive(lm, prompt, n_tok, "greedy", run_rng(seed))
        assert toks == ar, name
        out.append(dict(name=name, model=mc.to_dict(), seed=seed, deep_scale=deep_scale, deep_from=8,
                        cfg=cfgkw, prompt=prompt, max_tokens=n_tok, tokens=toks, exit_head="layer",
                        metrics=metrics_list(m), trace_csv=trace_text(tr), min_margins=lm.margin_report()))
        print(name, metrics_list(m), flush=True)
    return out


SAMPLING_CASES = [
    ("s_b1", 32, 16, 0, 1.0, dict(n_layers=32, exit_depth=8), None, 128),
    ("s_b0", 32, 16, 4, 0.0, dict(n_layers=32, exit_depth=8), [1], 64),
    ("s_b2", 32, 16, 12, 2.0, dict(n_layers=32, exit_depth=8), [11, 4, 4, 0], 96),
    ("s_deep_exit", 32, 16, 5, 1.0, dict(n_layers=32, exit_depth=8, exit_stage=2), [6, 6], 64),
    ("s_comm_lat", 32, 16, 6, 1.5, dict(n_layers=32, exit_depth=8, comm_latency=1), [2, 7], 64),
    ("s_remainder", 33, 16, 7, 0.7, dict(n_layers=33, exit_depth=8), [9, 0, 2], 80),
    ("s_v1000", 32, 1000, 10, 0.5, dict(n_layers=32, exit_depth=8), [17, 999, 0], 64),
]


def make_sampling():
    out = []
    for name, n, vocab, seed, beta, cfgkw, prompt, max_tokens in SAMPLING_CASES:
        lm = sp.ToyLM(n_layers=n, vocab=vocab, seed=sp.derive_seed(seed, "lm"), misalignment=beta)
        cfg = sp.PipelineConfig(**cfgkw)
        if prompt is None:
            prompt = sp.default_prompt(vocab, run_rng(seed))
        toks, m, tr = sp.decode_ppsd(lm, cfg, prompt, max_tokens, "sampling", run_rng(seed))
        ar = sp.decode_autoregressive(lm, prompt, max_tokens, "sampling", run_rng(seed))
        fr, fm, _ = sp.decode_ppsd(lm, cfg, prompt, max_tokens, "sampling", run_rng(seed), force_reject=True)
        assert fr == ar
        out.append(dict(name=name, n_layers=n, vocab=vocab, lm_seed=lm.seed, beta=beta, cfg=cfgkw,
                        prompt=list(map(int, prompt)), max_tokens=max_tokens, rng_seed=run_rng(seed).seed,
                        tokens=toks, metrics=metrics_list(m), trace_csv=trace_text(tr), ar_tokens=ar,
                        force_reject_metrics=metrics_list(fm)))
    # simulate_ppsd with a toy sampling oracle (default prompt from the run stream)
    for seed, beta in ((1, 1.0), (2, 0.5)):
        lm = sp.ToyLM(n_layers=32, vocab=16, seed=sp.derive_seed(seed, "lm"), misalignment=beta)
        tr = EventTrace()
        m = sp.simulate_ppsd(sp.PipelineConfig(32, 8), sp.AcceptanceOracle.toylm_sampling(lm), 100,
                             run_rng(seed), trace=tr)
        out.append(dict(name=f"sim_sampling_{seed}", kind="simulate", n_layers=32, vocab=16, lm_seed=lm.seed,
                        beta=beta, cfg=dict(n_layers=32, exit_depth=8), rng_seed=run_rng(seed).seed,
                        max_tokens=100, metrics=metrics_list(m), trace_csv=trace_text(tr)))
    return out


EESD_SAMPLING = [  # (lm seed, beta, cfg kwargs, gamma, horizon)
    (1, 1.0, dict(n_layers=32, exit_depth=8), 3, 80),
    (2, 0.5, dict(n_layers=32, exit_depth=8), 5, 100),
    (3, 2.0, dict(n_layers=32, exit_depth=8), 8, 64),
    (4, 1.0, dict(n_layers=32, exit_depth=8, exit_stage=2), 4, 60),
    (5, 0.8, dict(n_layers=33, exit_depth=8, comm_latency=1), 6, 70),
    (6, 0.0, dict(n_layers=16, exit_depth=4), 5, 50),
]


def make_eesd_sampling():
    out = []
    for seed, beta, cfgkw, gamma, horizon in EESD_SAMPLING:
        lm = sp.ToyLM(n_layers=cfgkw["n_layers"], vocab=16, seed=sp.derive_seed(seed, "lm"), misalignment=beta)
        tr = EventTrace()
        m = sp.simulate_eesd(sp.PipelineConfig(**cfgkw), gamma, sp.AcceptanceOracle.toylm_sampling(lm), horizon,
                             run_rng(seed), trace=tr)
        out.append(dict(lm_seed=lm.seed, n_layers=cfgkw["n_layers"], vocab=16, beta=beta, cfg=cfgkw, gamma=gamma,
                        horizon=horizon, rng_seed=run_rng(seed).seed, metrics=metrics_list(m),
                        trace_csv=trace_text(tr)))
    return out


HARNESS_RUNS = [
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=128, oracle="bernoulli", alpha=0.7, seed=1),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=96, oracle="toylm-greedy", beta=1.0, seed=2),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=96, oracle="toylm-sampling", beta=0.5, seed=3),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=64, exit_stage=2, oracle="toylm-greedy",
         beta=1.5, seed=4),
    dict(regime="ppsd", n_layers=33, exit_depth=8, horizon=80, comm_latency=1, oracle="bernoulli",
         alpha=0.55, seed=5, steady_state=True),
    dict(regime="eesd", n_layers=32, exit_depth=8, horizon=100, gamma=5, oracle="bernoulli", alpha=0.6,
         seed=6),
    dict(regime="eesd", n_layers=32, exit_depth=8, horizon=100, gamma=3, oracle="toylm-greedy", beta=1.0,
         seed=7),
    dict(regime="eesd", n_layers=32, exit_depth=8, horizon=60, gamma=4, exit_stage=2, oracle="bernoulli",
         alpha=0.8, seed=8),
    dict(regime="autoregressive", n_layers=32, exit_depth=8, horizon=50, seed=9),
    dict(regime="autoregressive", n_layers=24, exit_depth=5, horizon=20, comm_latency=2, seed=10,
         steady_state=True),
    dict(regime="ppsd", n_layers=16, exit_depth=4, horizon=64, oracle="toylm-greedy", beta=0.0, vocab=64,
         seed=11),
    dict(regime="eesd", n_layers=32, exit_depth=8, horizon=80, gamma=4, oracle="toylm-sampling", beta=0.7,
         seed=12),
]
HARNESS_BAD = [
    dict(regime="nope", n_layers=32, exit_depth=8, horizon=10),
    dict(regime="ppsd", n_layers=32, exit_depth=40, horizon=10, oracle="bernoulli", alpha=0.5),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=0, oracle="bernoulli", alpha=0.5),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, exit_stage=4, oracle="bernoulli", alpha=0.5),
    dict(regime="autoregressive", n_layers=32, exit_depth=8, horizon=10, gamma=3),
    dict(regime="autoregressive", n_layers=32, exit_depth=8, horizon=10, beta=0.5),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="magic"),
    dict(regime="eesd", n_layers=32, exit_depth=8, horizon=10, oracle="bernoulli", alpha=0.5),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, gamma=2, oracle="bernoulli", alpha=0.5),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="bernoulli"),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="bernoulli", alpha=1.5),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="bernoulli", alpha=0.5, beta=1.0),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="toylm-greedy", alpha=0.5),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="toylm-greedy", beta=-1.0),
    dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="toylm-greedy", vocab=1),
    dict(regime="ppsd", n_layers=32.0, exit_depth=8, horizon=10, oracle="bernoulli", alpha=0.5),
    dict(regime="ppsd", n_layers=8, exit_depth=8, horizon=10, exit_stage=1, oracle="bernoulli", alpha=0.5),
]


def make_harness():
    from specpipe import harness as H

    runs = []
    for kw in HARNESS_RUNS:
        res = H.run(H.ExperimentConfig(**kw), want_trace=True)
        runs.append(dict(config=kw, row=H.result_row(res), measured_alpha=res.measured_alpha,
                         trace_csv=trace_text(res.trace)))
    bad = []
    for kw in HARNESS_BAD:
        try:
            H.ExperimentConfig(**kw)
            bad.append(dict(config=kw, error=None))
        except H.ConfigError as exc:
            bad.append(dict(config=kw, field=exc.field, error=str(exc)))
    align = []
    for seed, beta, vocab, n, e in ((0, 1.0, 16, 32, 8), (3, 0.3, 16, 32, 4), (5, 2.0, 64, 24, 12), (9, 0.0, 16, 8, 2)):
        lm = sp.ToyLM(n_layers=n, vocab=vocab, seed=sp.derive_seed(seed, "lm"), misalignment=beta)
        align.append(dict(n_layers=n, vocab=vocab, lm_seed=lm.seed, beta=beta, exit_depth=e,
                          empirical_alpha=lm.empirical_alpha(e, 200), greedy_agreement=lm.greedy_agreement(e, 200),
                          empirical_alpha_seeded=lm.empirical_alpha(e, 37, eval_seed=12345)))
    reports = [dict(args=[a, g, n, e], text=H.analytic_report(a, g, n, e))
               for a, g, n, e in ((0.7, 4, 32, 8), (1.0, 5, 32, 8), (0.0, 1, 40, 20), (0.55, 10, 80, 10))]
    sweep = H.SweepSpec.from_dict(dict(base=dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=48,
                                                 oracle="bernoulli", alpha=0.5, seed=3),
                                       axes={"alpha": [0.3, 0.9], "exit_depth": [4, 8]}))
    buf = io.StringIO()
    H.write_results_csv(H.sweep(sweep), buf)
    return [dict(kind="runs", cases=runs), dict(kind="bad", cases=bad), dict(kind="align", cases=align),
            dict(kind="report", cases=reports), dict(kind="sweep", csv=buf.getvalue())]


CLI_HARNESS = [
    ["analytic", "--alpha", "0.7", "--gamma", "4", "--n-layers", "32", "--exit-depth", "8"],
    ["analytic", "--alpha", "0.4", "--gamma", "6", "--n-layers", "40", "--exit-depth", "10", "--t-draft", "0.3"],
    ["run", "--regime", "ppsd", "--n-layers", "32", "--exit-depth", "8", "--horizon", "64", "--oracle",
     "bernoulli", "--alpha", "0.6", "--seed", "4"],
    ["run", "--regime", "ppsd", "--n-layers", "32", "--exit-depth", "8", "--horizon", "64", "--oracle",
     "toylm-greedy", "--beta", "1.0", "--seed", "2"],
    ["run", "--regime", "eesd", "--n-layers", "32", "--exit-depth", "8", "--horizon", "50", "--gamma", "4",
     "--oracle", "toylm-greedy", "--beta", "0.5", "--steady-state"],
    ["run", "--regime", "autoregressive", "--n-layers", "32", "--exit-depth", "8", "--horizon", "20"],
    ["run", "--config", "{config_json}", "--horizon", "40"],
    ["run", "--config", "{config_json}", "--dump-config"],
    ["run", "--regime", "ppsd", "--n-layers", "32", "--exit-depth", "8", "--horizon", "10"],
    ["run", "--regime", "ppsd", "--n-layers", "32", "--exit-depth", "8", "--horizon", "10", "--oracle",
     "bernoulli", "--alpha", "2.0"],
    ["trace", "--regime", "ppsd", "--n-layers", "32", "--exit-depth", "8", "--horizon", "10", "--oracle",
     "bernoulli", "--alpha", "0.5"],
    ["sweep", "--config", "{sweep_json}"],
]
CLI_CONFIG = dict(regime="ppsd", n_layers=24, exit_depth=6, horizon=30, oracle="toylm-sampling", beta=0.8, seed=5)
CLI_SWEEP = dict(base=dict(regime="eesd", n_layers=32, exit_depth=8, horizon=40, gamma=3, oracle="bernoulli",
                           alpha=0.5, seed=2), axes={"gamma": [2, 5], "alpha": [0.25, 0.75]})


CLI_DECODE = [["decode", "--n-layers", "32", "--exit-depth", "8", "--beta", "1.0", "--mode", "greedy", "--max-tokens", "48", "--check-ar"], ["decode", "--n-layers", "32", "--exit-depth", "8", "--beta", "1.0", "--max-tokens", "48", "--seed", "3"], ["decode", "--n-layers", "33", "--exit-depth", "8", "--beta", "2.0", "--mode", "sampling", "--max-tokens", "40", "--prompt", "1,2,3", "--force-reject", "--check-ar"], ["decode", "--n-layers", "32", "--exit-depth", "8", "--exit-stage", "2", "--comm-latency", "1", "--beta", "0.5", "--mode", "greedy", "--max-tokens", "32"]]


def make_cli_decode():
    import subprocess

    env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src")
    out = []
    for argv in CLI_DECODE:
        r = subprocess.run([sys.executable, "-m", "specpipe.cli", *argv], capture_output=True, text=True, env=env,
                           cwd="/tmp", timeout=600)
        out.append(dict(argv=argv, stdout=r.stdout, returncode=r.returncode))
    return out


def make_cli_harness():
    import subprocess
    import tempfile

    out = []
    with tempfile.TemporaryDirectory() as d:
        paths = {"config_json": os.path.join(d, "config.json"), "sweep_json": os.path.join(d, "sweep.json")}
        with open(paths["config_json"], "w") as fh:
            fh.write(json.dumps(CLI_CONFIG))
        with open(paths["sweep_json"], "w") as fh:
            fh.write(json.dumps(CLI_SWEEP))
        env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src")
        for argv in CLI_HARNESS:
            real = [a.format(**paths) for a in argv]
            r = subprocess.run([sys.executable, "-m", "specpipe.cli", *real], capture_output=True, text=True,
                               env=env, cwd=d, timeout=600)
            out.append(dict(argv=argv, stdout=r.stdout, stderr=r.stderr, returncode=r.returncode))
    # file texts, not dicts: the fixture is dumped with sorted keys and the
    # sweep axes' order is significant
    return [dict(config_json=json.dumps(CLI_CONFIG), sweep_json=json.dumps(CLI_SWEEP), commands=out)]


def main(argv):
    which = set(argv[1:]) or {"toy", "bern", "acc", "eesd", "tf", "samp", "harness", "cli", "clidec", "eesdsamp",
                              "tfhead"}
    jobs = [("toy", "toylm_decode.json", make_toy), ("bern", "bernoulli.json", make_bernoulli),
            ("acc", "acceptance200.json", make_acceptance200), ("eesd", "eesd_toy.json", make_eesd),
            ("tf", "transformer.json", make_transformer), ("samp", "toylm_sampling.json", make_sampling),
            ("harness", "harness.json", make_harness), ("cli", "cli_harness.json", make_cli_harness),
            ("clidec", "cli_decode.json", make_cli_decode), ("eesdsamp", "eesd_sampling.json", make_eesd_sampling),
            ("tfhead", "transformer_head.json", make_transformer_head)]
    for key, fname, fn in jobs:
        if key in which:
            data = dict(reference="specpipe " + sp.__version__, generator="tests/golden/make_golden.py",
                        cases=fn())
            with open(os.path.join(HERE, fname), "w") as fh:
                json.dump(data, fh, indent=0, sort_keys=True)
            print("wrote", fname, len(data["cases"]), "cases")


if __name__ == "__main__":
    main(sys.argv)
