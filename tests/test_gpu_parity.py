"""GPU parity: the sm_100a engine (through the C ABI) against the pinned oracle.

Every comparison is against fixtures produced by the real reference
(tests/golden/*.json) or against the CPU oracle on identical weights.
Integer outputs (tokens, accept/reject counts, ticks, trace rows) must be
bit-exact; logits must agree within the tolerance stated in each test.
"""

import hashlib

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

ppsd = pytest.importorskip("paper_2509_19368_b200")


def _metrics_list(m):
    return [m.committed_tokens, m.ticks, m.accepts, m.rejects, m.alpha_all_measured,
            m.throughput, m.speedup_vs_ar]


def _cfg(d):
    return ppsd.PipelineConfig(d["n_layers"], d["exit_depth"], exit_stage=d.get("exit_stage"),
                               comm_latency=d.get("comm_latency", 0))


# ---------------------------------------------------------------- ToyLM ----

@pytest.mark.parametrize("case", load_golden("toylm_decode.json"), ids=lambda c: c["name"])
def test_toylm_decode_bit_exact(case):
    lm = ppsd.ToyLM(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    cfg = _cfg(case["cfg"])
    rng = ppsd.RngStream(case["rng_seed"])
    toks, m, tr = ppsd.decode_ppsd(lm, cfg, case["prompt"], case["max_tokens"], "greedy", rng)
    assert toks == case["tokens"]
    assert _metrics_list(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]
    ar = ppsd.decode_autoregressive(lm, case["prompt"], case["max_tokens"], "greedy", rng)
    assert ar == case["ar_tokens"]
    if case["max_tokens"]:
        _, mf, _ = ppsd.decode_ppsd(lm, cfg, case["prompt"], case["max_tokens"], "greedy", rng,
                                    force_reject=True)
        assert _metrics_list(mf) == case["force_reject_metrics"]


def test_toylm_acceptance200_bit_exact():
    cfg = ppsd.PipelineConfig(32, 8)
    for i, case in enumerate(load_golden("acceptance200.json")):
        lm = ppsd.ToyLM(32, 16, case["lm_seed"], 1.0)
        toks, m, _ = ppsd.decode_ppsd(lm, cfg, case["prompt"], 256, "greedy", ppsd.RngStream(i))
        assert hashlib.sha256(",".join(map(str, toks)).encode()).hexdigest() == case["tokens_sha256"], i
        assert _metrics_list(m) == case["metrics"], i


@pytest.mark.parametrize("case", load_golden("bernoulli.json"), ids=lambda c: f"a{c['alpha']}-{c['horizon']}")
def test_bernoulli_schedule_bit_exact(case):
    cfg = _cfg(case["cfg"])
    tr = ppsd.EventTrace()
    m = ppsd.simulate_ppsd(cfg, ppsd.AcceptanceOracle.bernoulli(case["alpha"]), case["horizon"],
                           ppsd.RngStream(case["rng_seed"]), trace=tr)
    assert _metrics_list(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]


def test_input_validation_matches_reference():
    lm = ppsd.ToyLM(32, 16, 1, 1.0)
    cfg = ppsd.PipelineConfig(32, 8)
    rng = ppsd.RngStream(0)
    with pytest.raises(ValueError):
        ppsd.decode_ppsd(lm, ppsd.PipelineConfig(24, 8), [1], 4, "greedy", rng)
    with pytest.raises(ValueError):
        ppsd.decode_ppsd(lm, cfg, [], 4, "greedy", rng)
    with pytest.raises(ValueError):
        ppsd.decode_ppsd(lm, cfg, [16], 4, "greedy", rng)
    with pytest.raises(ValueError):
        ppsd.decode_ppsd(lm, cfg, [1], 4, "argmax", rng)
    toks, m, tr = ppsd.decode_ppsd(lm, cfg, [1], 0, "greedy", rng)
    assert toks == [] and m.committed_tokens == 0 and m.ticks == 0 and len(tr) == 0


# ---------------------------------------------------------- transformer ----

@pytest.fixture(scope="module")
def tiny_models():
    cache = {}

    def get(seed, deep_scale, deep_from=8):
        key = (seed, deep_scale, deep_from)
        if key not in cache:
            cache[key] = ppsd.TransformerLM(ppsd.TransformerConfig.tiny(), seed=seed,
                                            deep_scale=deep_scale, deep_from=deep_from)
        return cache[key]

    return get


@pytest.mark.parametrize("schedule", ["pipelined", "folded"])
@pytest.mark.parametrize("case", load_golden("transformer.json"), ids=lambda c: c["name"])
def test_tiny_transformer_matches_reference_scheduler(case, schedule, tiny_models):
    """The reference's decode_ppsd driving the fp64 CPU decoder produced these
    tokens, accept/reject counts and trace; the GPU engine must match exactly,
    under both single-device schedules."""
    lm = tiny_models(case["seed"], case["deep_scale"], case["deep_from"])
    cfg = _cfg(case["cfg"])
    lm.schedule = schedule
    try:
        toks, m, tr = ppsd.decode_ppsd(lm, cfg, case["prompt"], case["max_tokens"], "greedy",
                                       ppsd.RngStream(0))
        assert ppsd.engine_for(lm, cfg).schedule("greedy") == schedule
    finally:
        lm.schedule = "auto"
    assert toks == case["tokens"]
    assert _metrics_list(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]
    assert ppsd.decode_autoregressive(lm, case["prompt"], case["max_tokens"], "greedy",
                                      ppsd.RngStream(0)) == case["tokens"]


def _oracle_for(config, seed, deep_scale, deep_from):
    from oracle.transformer import ModelShape, TransformerOracle

    shape = ModelShape(config.n_layers, config.d_model, config.n_heads, config.n_kv_heads,
                       config.head_dim, config.ffn_dim, config.vocab, config.rms_eps,
                       config.rope_theta)
    return TransformerOracle(shape, seed=seed, deep_scale=deep_scale, deep_from=deep_from,
                             max_ctx=config.max_ctx, threads=16)


SHAPES = {
    # the kernel instantiations of Llama-2-7B/13B/70B layers, at 2 layers each
    "l7b_2layer": dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=32, head_dim=128,
                       ffn_dim=11008, vocab=32000),
    "l13b_2layer": dict(n_layers=2, d_model=5120, n_heads=40, n_kv_heads=40, head_dim=128,
                        ffn_dim=13824, vocab=32000),
    "l70b_2layer": dict(n_layers=2, d_model=8192, n_heads=64, n_kv_heads=8, head_dim=128,
                        ffn_dim=28672, vocab=32000),
    "mid_gqa": dict(n_layers=4, d_model=1024, n_heads=16, n_kv_heads=4, head_dim=64,
                    ffn_dim=2816, vocab=4096),
}


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("kv", ["fp32", "bf16"])
def test_teacher_forced_logits_vs_oracle(name, kv):
    """Final-head logits after a 70-token prompt (spans two KV pages).
    Tolerance: fp32 KV |dz| <= 2e-4 * max|z| + 2e-4; bf16 KV 2e-2 * max|z| + 2e-2
    (bf16 rounding of K/V is the only extra error source)."""
    sh = SHAPES[name]
    config = ppsd.TransformerConfig(**sh, kv_dtype=kv, max_ctx=256)
    lm = ppsd.TransformerLM(config, seed=3, deep_scale=0.5, deep_from=1)
    rng = np.random.default_rng(5)
    prompt = [int(t) for t in rng.integers(0, config.vocab, size=70)]
    cfg = ppsd.PipelineConfig(config.n_layers, 1)
    eng = ppsd.engine_for(lm, cfg)
    eng.decode_ar(prompt, 1)
    got = eng.read_logits(1).astype(np.float64)
    orc = _oracle_for(config, 3, 0.5, 1)
    want = orc.logits_for_prefix(prompt)
    scale = np.abs(want).max()
    tol = (2e-4 if kv == "fp32" else 2e-2) * (scale + 1.0)
    err = np.abs(got - want).max()
    assert err <= tol, f"{name}/{kv}: max |dz| {err:.3e} > {tol:.3e}"
    if kv == "fp32":
        top2 = np.sort(want)[-2:]
        if top2[1] - top2[0] > 4 * tol:
            assert int(np.argmax(got)) == int(np.argmax(want))


@pytest.mark.parametrize("name", ["l7b_2layer", "mid_gqa"])
def test_ppsd_equals_ar_bit_exact(name):
    """Lossless greedy PPSD on the GPU: token-for-token equal to GPU AR (same
    kernels, deterministic reductions), several stage splits."""
    sh = dict(SHAPES[name])
    sh["n_layers"] = 8
    config = ppsd.TransformerConfig(**sh, kv_dtype="bf16", max_ctx=512)
    lm = ppsd.TransformerLM(config, seed=11, deep_scale=0.3, deep_from=2)
    prompt = [int(t) for t in np.random.default_rng(1).integers(0, config.vocab, size=20)]
    ar = ppsd.decode_autoregressive(lm, prompt, 96, "greedy", ppsd.RngStream(0))
    for e, k in ((2, 1), (4, 1), (3, 1), (2, 2)):
        cfg = ppsd.PipelineConfig(8, e, exit_stage=k)
        toks, m, tr = ppsd.decode_ppsd(lm, cfg, prompt, 96, "greedy", ppsd.RngStream(0))
        assert toks == ar, (e, k)
        assert m.committed_tokens == 96 and m.accepts + m.rejects == 96
        rows = [r for r in tr if r.kind in ("FINAL_TOKEN", "CHECK_TOKEN")]
        assert [r.token for r in rows] == toks


@pytest.mark.parametrize("name", ["l7b_2layer", "mid_gqa"])
def test_folded_equals_pipelined(name):
    """The folded single-device schedule (eager shallow stages, batched deep
    verdicts) returns exactly the pipelined schedule's tokens, metrics and
    trace — remainder stages, exit_stage > 1 and comm_latency included."""
    sh = dict(SHAPES[name])
    sh["n_layers"] = 10
    config = ppsd.TransformerConfig(**sh, kv_dtype="bf16", max_ctx=512)
    lm = ppsd.TransformerLM(config, seed=5, deep_scale=0.35, deep_from=2)
    prompt = [int(t) for t in np.random.default_rng(2).integers(0, config.vocab, size=21)]
    for e, k, cl in ((2, 1, 0), (3, 1, 0), (4, 1, 1), (2, 2, 0), (3, 3, 0), (2, 1, 2)):
        cfg = ppsd.PipelineConfig(10, e, exit_stage=k, comm_latency=cl)
        out = {}
        for sched in ("pipelined", "folded"):
            lm.schedule = sched
            toks, m, tr = ppsd.decode_ppsd(lm, cfg, prompt, 80, "greedy", ppsd.RngStream(0))
            eng = ppsd.engine_for(lm, cfg)
            assert eng.schedule("greedy") == sched
            out[sched] = (toks, _metrics_list(m), tr.to_csv())
            assert eng.last["schedule"] == sched
        lm.schedule = "auto"
        assert out["folded"] == out["pipelined"], (e, k, cl)


# ---------------------------------------------------------------- EESD -----

@pytest.mark.parametrize("case", load_golden("eesd_toy.json"), ids=lambda c: f"{c['kind']}-g{c['gamma']}")
def test_eesd_matches_reference(case):
    cfg = ppsd.PipelineConfig(32, 8)
    tr = ppsd.EventTrace()
    if case["kind"] == "toy":
        lm = ppsd.ToyLM(32, 16, case["lm_seed"], case["beta"])
        oracle = ppsd.AcceptanceOracle.toylm_greedy(lm)
    else:
        oracle = ppsd.AcceptanceOracle.bernoulli(case["alpha"])
    m = ppsd.simulate_eesd(cfg, case["gamma"], oracle, case["horizon"], ppsd.RngStream(case["rng_seed"]), trace=tr)
    assert _metrics_list(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]


@pytest.mark.parametrize("gamma,seed,ds", [(5, 0, 0.1), (3, 1, 0.25), (10, 2, 0.15)])
def test_tiny_transformer_eesd_matches_oracle(gamma, seed, ds, tiny_models):
    """GPU EESD (batched verify through kMatHeadV) vs the oracle port's
    simulate_eesd (pinned to reference EESD goldens) on the CPU decoder."""
    from oracle import specpipe_port as sp
    from oracle.transformer import TransformerOracle, tiny_config

    lm = tiny_models(seed, ds)
    prompt = ppsd.default_prompt(256, ppsd.RngStream(seed))
    toks, m, tr = ppsd.decode_eesd(lm, ppsd.PipelineConfig(32, 8), prompt, 96, gamma)
    orc = TransformerOracle(tiny_config(), seed=seed, deep_scale=ds, deep_from=8)
    want_toks, want_m, rows = sp.simulate_eesd(orc, 32, 8, gamma, 96, 0, prompt=prompt)
    assert toks == want_toks[:len(toks)]
    assert _metrics_list(m) == list(want_m)
    assert tr.to_csv() == sp.trace_csv(rows)


@pytest.mark.parametrize("gamma", [1, 4, 7, 15])
def test_eesd_lossless_vs_ar(gamma):
    config = ppsd.TransformerConfig(6, 512, 8, 2, 64, 1408, 2048, kv_dtype="bf16", max_ctx=512)
    lm = ppsd.TransformerLM(config, seed=21, deep_scale=0.3, deep_from=2)
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, config.vocab, size=40)]
    ar = ppsd.decode_autoregressive(lm, prompt, 100, "greedy", ppsd.RngStream(0))
    toks, m, _ = ppsd.decode_eesd(lm, ppsd.PipelineConfig(6, 2), prompt, 100, gamma)
    assert toks[:100] == ar
    assert m.committed_tokens >= 100


def test_folded_edge_cases():
    """Folded ≡ pipelined on the edges: one-token prompt (no prefill), one
    generated token, force_reject (every verdict a rollback), a context that
    crosses a KV page inside a deep batch, max_ctx-bound runs."""
    sh = dict(SHAPES["mid_gqa"])
    sh["n_layers"] = 8
    config = ppsd.TransformerConfig(**sh, kv_dtype="bf16", max_ctx=200)
    lm = ppsd.TransformerLM(config, seed=9, deep_scale=0.4, deep_from=2)
    cfg = ppsd.PipelineConfig(8, 2)
    cases = [([5], 30, False), ([3, 1, 4], 1, False), ([2, 7], 40, True), (list(range(60)), 40, False),
             ([11] * 3, 200 - 3 - cfg.n_stages * cfg.hop_period - 2, False)]
    for prompt, n, fr in cases:
        out = {}
        for sched in ("pipelined", "folded"):
            lm.schedule = sched
            toks, m, tr = ppsd.decode_ppsd(lm, cfg, prompt, n, "greedy", ppsd.RngStream(0), force_reject=fr)
            out[sched] = (toks, _metrics_list(m), tr.to_csv())
        lm.schedule = "auto"
        assert out["folded"] == out["pipelined"], (len(prompt), n, fr)
        assert out["folded"][0] == ppsd.decode_autoregressive(lm, prompt, n, "greedy", ppsd.RngStream(0))
    with pytest.raises(ValueError):
        ppsd.decode_ppsd(lm, cfg, [1, 2], 200, "greedy", ppsd.RngStream(0))


# ------------------------------------------------ decoder-layer exit head --

@pytest.mark.parametrize("schedule", ["pipelined", "folded"])
@pytest.mark.parametrize("case", load_golden("transformer_head.json"), ids=lambda c: c["name"])
def test_head_layer_matches_reference_scheduler(case, schedule):
    """Exit head = one decoder layer (own KV) + norm head, the paper's main
    configuration: the reference decode_ppsd driving the fp64 oracle with that
    head produced these tokens / counts / traces; the GPU matches exactly."""
    lm = ppsd.TransformerLM(ppsd.TransformerConfig.tiny(), seed=case["seed"], deep_scale=case["deep_scale"],
                            deep_from=case["deep_from"], exit_head="layer")
    cfg = _cfg(case["cfg"])
    lm.schedule = schedule
    toks, m, tr = ppsd.decode_ppsd(lm, cfg, case["prompt"], case["max_tokens"], "greedy", ppsd.RngStream(0))
    assert toks == case["tokens"]
    assert _metrics_list(m) == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]


@pytest.mark.parametrize("name", ["l7b_2layer", "mid_gqa"])
def test_head_layer_lossless_and_schedules_agree(name):
    """With the decoder-layer exit head: folded ≡ pipelined (tokens, metrics,
    trace), PPSD ≡ AR and EESD ≡ AR token-for-token (the tcgen05 prefill also
    fills the head layer's KV for the prompt)."""
    sh = dict(SHAPES[name])
    sh["n_layers"] = 8
    config = ppsd.TransformerConfig(**sh, kv_dtype="bf16", max_ctx=512)
    lm = ppsd.TransformerLM(config, seed=13, deep_scale=0.3, deep_from=2, exit_head="layer")
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, config.vocab, size=40)]
    ar = ppsd.decode_autoregressive(lm, prompt, 64, "greedy", ppsd.RngStream(0))
    for e, k, cl in ((2, 1, 0), (2, 2, 0), (4, 1, 1)):
        cfg = ppsd.PipelineConfig(8, e, exit_stage=k, comm_latency=cl)
        out = {}
        for sched in ("pipelined", "folded"):
            lm.schedule = sched
            toks, m, tr = ppsd.decode_ppsd(lm, cfg, prompt, 64, "greedy", ppsd.RngStream(0))
            out[sched] = (toks, _metrics_list(m), tr.to_csv())
        lm.schedule = "auto"
        assert out["folded"] == out["pipelined"], (e, k, cl)
        assert out["folded"][0] == ar, (e, k, cl)
        assert 0 < out["folded"][1][2] < 64  # accepts and rejects both occur
    et, em, _ = ppsd.decode_eesd(lm, ppsd.PipelineConfig(8, 2), prompt, 64, 3)
    assert et[:64] == ar
