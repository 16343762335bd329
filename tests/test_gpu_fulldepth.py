"""Full-depth parity at the BENCHMARKED configuration (BASELINE config 2).

The bench decodes 512 tokens of a Llama-2-7B-shaped model (32 layers, d 4096,
V 32000, bf16 weights, bf16 KV cache) with exit E=8 (4 stages), deep_scale
0.08, a 128-token prompt prefilled by the tcgen05 GEMM, under the folded
schedule. This test runs exactly that decode on the GPU with the logits tap
on (ppsd_set_logits_tap: the exit and final logits each verdict / draft
used, by position) and checks it against the CPU oracle
(oracle/transformer.py, fp32 numpy, K/V rounded to bf16 as the GPU stores
them) teacher-forced along the GPU's own token path:

* logits: every position's exit-head and final-head rows, |dz| <= TOL_REL *
  (max|z| + 1) with TOL_REL below (fp32 accumulation-order differences over
  32 layers + bf16-rounding flips of K/V elements near a rounding boundary);
* tokens (margin-aware, reference semantics speccore.py:116-126): where the
  oracle's final-head top-1/top-2 margin exceeds 4*tol the GPU token is the
  oracle argmax; inside the margin it is within 2*tol of the max;
* verdicts: where both heads' margins are clear, accept <=> exit argmax ==
  final argmax (greedy_match, pipesim.py:351-358), position by position from
  the trace, so the accepted-token count is pinned too;
* trace invariants: the reference's work-conservation, commit-order and
  flush-discipline checkers (pkg/tests/helpers.py:80-151, tests/trace_checks.py)
  hold on the 512-token trace.

The margin histogram is printed (and written to $PPSD_PARITY_OUT as JSON:
profiles/r02_fulldepth_parity.json).
"""

import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ppsd = pytest.importorskip("paper_2509_19368_b200")

TOL_REL = 1e-3


def _run_gpu(config, cfg, prompt, n_new, deep_scale, exit_depth, seed):
    import torch

    lm = ppsd.TransformerLM(config, seed=seed, deep_scale=deep_scale, deep_from=exit_depth)
    eng = ppsd.engine_for(lm, cfg)
    tap = torch.full((n_new + 1, 2, config.vocab), float("nan"), dtype=torch.float32, device=lm.device)
    eng.set_logits_tap(tap)
    try:
        toks, m, tr = eng.decode(prompt, n_new)
    finally:
        eng.set_logits_tap(None)
    sched = eng.last["schedule"]
    out = tap.cpu().numpy().astype(np.float64)
    del tap, eng, lm
    torch.cuda.empty_cache()
    return toks, m, tr, sched, out


def test_bench_config_full_depth_vs_oracle():
    import bench
    from oracle.transformer import ModelShape, TransformerOracle

    config = ppsd.TransformerConfig.llama2_7b(max_ctx=1024)
    E, n_new = bench.EXIT_DEPTH, bench.NEW_TOKENS
    cfg = ppsd.PipelineConfig(config.n_layers, E)
    prompt = bench.bench_prompt(config.vocab)
    toks, m, tr, sched, tap = _run_gpu(config, cfg, prompt, n_new, bench.DEEP_SCALE, E, bench.SEED)
    assert sched == "folded"  # the bench's schedule
    assert m.committed_tokens == n_new
    # the reference's trace invariants (pkg/tests/helpers.py:80-151) on the bench trace
    from trace_checks import check_all

    check_all(tr, cfg.n_stages, cfg.exit_stage)

    shape = ModelShape(config.n_layers, config.d_model, config.n_heads, config.n_kv_heads, config.head_dim,
                       config.ffn_dim, config.vocab, config.rms_eps, config.rope_theta)
    orc = TransformerOracle(shape, seed=bench.SEED, deep_scale=bench.DEEP_SCALE, deep_from=E, dtype=np.float32,
                            max_ctx=config.max_ctx, threads=os.cpu_count() or 8, rope_fp32=True, kv_bf16=True)
    path = list(prompt) + list(toks[:-1])
    ze, zf = orc.path_logits(path, first=len(prompt) - 1, exit_layer=E)  # row i: position i + 1
    del orc

    report = {"config": "llama2-7b shape, 32 layers, E=8, deep_scale 0.08, bf16 KV, prompt 128, 512 tokens, "
                        "folded schedule, tcgen05 prefill", "tol_rel": TOL_REL,
              "trace_rows": len(list(tr)), "trace_invariants": "work conservation, commit order, flush discipline: ok"}
    # ---- logits, both heads, every position ----
    worst = {}
    for which, z_or in ((0, ze), (1, zf)):
        g = tap[1:, which, :]
        have = ~np.isnan(g).any(axis=1)
        assert have.sum() >= 16, f"head {which}: only {have.sum()} tapped positions"
        tol = TOL_REL * (np.abs(z_or).max(axis=1) + 1.0)
        err = np.abs(g - z_or).max(axis=1)
        ratio = np.where(have, err / tol, 0.0)
        name = ("exit", "final")[which]
        worst[name] = float(ratio.max())
        report[f"{name}_positions"] = int(have.sum())
        report[f"{name}_max_abs_err"] = float(np.where(have, err, 0.0).max())
        report[f"{name}_max_err_over_tol"] = float(ratio.max())
        bad = np.nonzero(ratio > 1.0)[0]
        assert bad.size == 0, f"{name} head: {bad.size} positions over tolerance, worst {ratio.max():.2f}x tol at {bad[:8] + 1}"

    # ---- tokens, margin-aware ----
    tolf = TOL_REL * (np.abs(zf).max(axis=1) + 1.0)
    top2 = np.sort(zf, axis=1)[:, -2:]
    marg = top2[:, 1] - top2[:, 0]
    am = zf.argmax(axis=1)
    t = np.asarray(toks)
    clear = marg > 4 * tolf
    assert clear.sum() >= 64
    mism = np.nonzero(clear & (t != am))[0]
    assert mism.size == 0, f"tokens differ from the oracle argmax at clear-margin positions {mism[:8] + 1}"
    near = ~clear
    zt = zf[np.arange(len(t)), t]
    assert np.all(zt[near] >= top2[near, 1] - 2 * tolf[near]), "near-tie token far from the oracle max"
    report["token_positions"] = int(len(t))
    report["token_clear_margin"] = int(clear.sum())
    report["token_equal_oracle_argmax"] = int((t == am).sum())

    # ---- verdicts (accepted-token count) ----
    tole = TOL_REL * (np.abs(ze).max(axis=1) + 1.0)
    te2 = np.sort(ze, axis=1)[:, -2:]
    clear_e = (te2[:, 1] - te2[:, 0]) > 4 * tole
    pred_accept = ze.argmax(axis=1) == am
    verdict = {}
    for r in tr:
        if r.kind in ("FINAL_TOKEN", "CHECK_TOKEN"):
            verdict[r.position] = r.kind == "FINAL_TOKEN"
    assert sorted(verdict) == list(range(1, n_new + 1))
    got_accept = np.array([verdict[p] for p in range(1, n_new + 1)])
    both = clear & clear_e
    vm = np.nonzero(both & (got_accept != pred_accept))[0]
    assert vm.size == 0, f"verdicts differ from the oracle's greedy_match at {vm[:8] + 1}"
    assert got_accept.sum() == m.accepts
    report["verdict_positions_checked"] = int(both.sum())
    report["accepts_gpu"] = int(m.accepts)
    report["accepts_oracle_predicted_all_positions"] = int(pred_accept.sum())

    # margin histogram (units of tol)
    edges = [0, 1, 4, 16, 64, 256, math.inf]
    hist = {}
    for name, mg, tl in (("final", marg, tolf), ("exit", te2[:, 1] - te2[:, 0], tole)):
        q = mg / tl
        hist[name] = {f"[{edges[i]},{edges[i + 1]})": int(((q >= edges[i]) & (q < edges[i + 1])).sum())
                      for i in range(len(edges) - 1)}
    report["margin_histogram_in_tol_units"] = hist
    print(json.dumps(report, indent=1))
    out = os.environ.get("PPSD_PARITY_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump(report, fh, indent=1)
