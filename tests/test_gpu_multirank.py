"""The multi-rank engine path (ppsd_step_*) on ONE GPU: 2 and 4 stage-range
engines in one process, boxes exchanged by device copies instead of NCCL.
Tokens, metrics and trace must equal the single-engine decode bit-for-bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ppsd = pytest.importorskip("paper_2509_19368_b200")


def run_loopback(shards, prompt, max_tokens, mode="greedy", seed=0, force_reject=False):
    import torch

    steps = [s.begin(prompt, max_tokens, force_reject, mode=mode, rng=ppsd.RngStream(seed)) for s in shards]
    assert len(set(steps)) == 1

    def exchange():
        torch.cuda.synchronize()
        boxes = torch.stack([s.outbox for s in shards])
        for s in shards:
            s.inbox.copy_(boxes)
        torch.cuda.synchronize()

    for _ in range(steps[0]):
        for s in shards:
            s.prefill_compute()
        exchange()
    committed = 0
    while True:
        for _ in range(max(1, max_tokens - committed)):
            for s in shards:
                s.compute()
            exchange()
            for s in shards:
                s.finish()
        polls = [s.poll() for s in shards]
        assert len(set(polls)) == 1, polls
        if polls[0][0]:
            break
        committed = polls[0][1]
    return [s.end() for s in shards]


@pytest.mark.parametrize("world,e", [(1, 2), (2, 2), (4, 2), (2, 3)])
def test_loopback_pipeline_equals_single_gpu(world, e):
    from paper_2509_19368_b200.distributed import StageShard

    config = ppsd.TransformerConfig(8, 512, 8, 8, 64, 1408, 2048, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, e)
    if world > cfg.n_stages:
        pytest.skip("more ranks than stages")
    prompt = [int(t) for t in np.random.default_rng(7).integers(0, config.vocab, size=21)]
    full = ppsd.TransformerLM(config, seed=5, deep_scale=0.3, deep_from=e)
    want_toks, want_m, want_tr = ppsd.decode_ppsd(full, cfg, prompt, 80, "greedy", ppsd.RngStream(0))
    shards = [StageShard(config, cfg, r, world, seed=5, deep_scale=0.3, deep_from=e) for r in range(world)]
    for toks, m, tr in run_loopback(shards, prompt, 80):
        assert toks == want_toks
        assert m == want_m
        assert tr.to_csv() == want_tr.to_csv()


@pytest.mark.parametrize("world,e,k", [(1, 2, 1), (2, 2, 1), (4, 2, 1), (2, 2, 2), (4, 2, 3)])
def test_loopback_decoder_layer_exit_head(world, e, k):
    """Table-1 exit head (a decoder layer before the exit norm) across ranks:
    only the exit stage's rank holds and runs it, prefill included."""
    from paper_2509_19368_b200.distributed import StageShard

    config = ppsd.TransformerConfig(8, 512, 8, 8, 64, 1408, 2048, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, e, exit_stage=k)
    prompt = [int(t) for t in np.random.default_rng(11).integers(0, config.vocab, size=19)]
    full = ppsd.TransformerLM(config, seed=6, deep_scale=0.3, deep_from=e, exit_head="layer")
    want_toks, want_m, want_tr = ppsd.decode_ppsd(full, cfg, prompt, 64, "greedy", ppsd.RngStream(0))
    shards = [StageShard(config, cfg, r, world, seed=6, deep_scale=0.3, deep_from=e, exit_head="layer")
              for r in range(world)]
    assert sum(s.lm.exit_layer_w is not None for s in shards) == 1  # the exit stage's rank
    for toks, m, tr in run_loopback(shards, prompt, 64):
        assert toks == want_toks
        assert m == want_m
        assert tr.to_csv() == want_tr.to_csv()


@pytest.mark.parametrize("world,e,k,head", [(2, 2, 1, "norm"), (2, 2, 2, "norm"), (4, 2, 3, "norm"),
                                             (2, 2, 1, "layer"), (4, 2, 3, "layer")])
def test_loopback_sampling_equals_single_gpu(world, e, k, head):
    """Sampling mode across ranks: the boxes carry the exit / final logits and
    every rank makes the same draft / verify / commit draws, so tokens,
    metrics and trace equal the single-device sampling decode."""
    from paper_2509_19368_b200.distributed import StageShard

    config = ppsd.TransformerConfig(8, 512, 8, 8, 64, 1408, 2048, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, e, exit_stage=k)
    prompt = [int(t) for t in np.random.default_rng(5).integers(0, config.vocab, size=15)]
    full = ppsd.TransformerLM(config, seed=8, deep_scale=0.3, deep_from=e, exit_head=head)
    want = ppsd.decode_ppsd(full, cfg, prompt, 48, "sampling", ppsd.RngStream(21))
    shards = [StageShard(config, cfg, r, world, seed=8, deep_scale=0.3, deep_from=e, exit_head=head)
              for r in range(world)]
    for toks, m, tr in run_loopback(shards, prompt, 48, mode="sampling", seed=21):
        assert toks == want[0]
        assert m == want[1]
        assert tr.to_csv() == want[2].to_csv()
    assert 0 < want[1].accepts < 48  # both verdicts occur
    # back to greedy on the same shards
    gt, gm, gtr = ppsd.decode_ppsd(full, cfg, prompt, 32, "greedy", ppsd.RngStream(0))
    for toks, m, tr in run_loopback(shards, prompt, 32):
        assert toks == gt and m == gm and tr.to_csv() == gtr.to_csv()


@pytest.mark.parametrize("mode,comm,force", [("greedy", 1, False), ("greedy", 0, True), ("sampling", 2, False),
                                            ("sampling", 0, True)])
def test_loopback_comm_latency_and_force_reject(mode, comm, force):
    """Hop latency (comm_latency ticks per stage boundary) and force_reject
    across ranks, greedy and sampling."""
    from paper_2509_19368_b200.distributed import StageShard

    config = ppsd.TransformerConfig(8, 512, 8, 8, 64, 1408, 2048, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, 2, comm_latency=comm)
    prompt = [int(t) for t in np.random.default_rng(17).integers(0, config.vocab, size=13)]
    full = ppsd.TransformerLM(config, seed=9, deep_scale=0.3, deep_from=2)
    want = ppsd.decode_ppsd(full, cfg, prompt, 32, mode, ppsd.RngStream(4), force_reject=force)
    shards = [StageShard(config, cfg, r, 2, seed=9, deep_scale=0.3, deep_from=2) for r in range(2)]
    for toks, m, tr in run_loopback(shards, prompt, 32, mode=mode, seed=4, force_reject=force):
        assert toks == want[0]
        assert m == want[1]
        assert tr.to_csv() == want[2].to_csv()


@pytest.mark.parametrize("n_prompt,max_tokens,mode", [(1, 1, "greedy"), (1, 9, "sampling"), (2, 1, "sampling"),
                                                      (3, 5, "greedy")])
def test_loopback_edge_lengths(n_prompt, max_tokens, mode):
    """One-token prompts (no prefill step), one-token decodes, both modes."""
    from paper_2509_19368_b200.distributed import StageShard

    config = ppsd.TransformerConfig(8, 512, 8, 8, 64, 1408, 2048, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, 2)
    prompt = [int(t) for t in np.random.default_rng(23).integers(0, config.vocab, size=n_prompt)]
    full = ppsd.TransformerLM(config, seed=3, deep_scale=0.3, deep_from=2)
    want = ppsd.decode_ppsd(full, cfg, prompt, max_tokens, mode, ppsd.RngStream(6))
    shards = [StageShard(config, cfg, r, 4, seed=3, deep_scale=0.3, deep_from=2) for r in range(4)]
    for toks, m, tr in run_loopback(shards, prompt, max_tokens, mode=mode, seed=6):
        assert toks == want[0]
        assert m == want[1]
        assert tr.to_csv() == want[2].to_csv()


@pytest.mark.parametrize("world,k,comm,force", [(2, 1, 0, False), (2, 2, 0, False), (4, 1, 0, False),
                                                (3, 1, 0, False), (2, 1, 1, False), (2, 1, 0, True),
                                                (4, 3, 0, False), (2, 6, 0, False), (4, 3, 1, True)])
def test_loopback_rank_fold(world, k, comm, force):
    """Per-rank fold (sched.h: sched_rfold_plan): 8 one-layer stages, so every
    rank with deferred stages and more than one stage batches them (eager exit
    stages when it owns k, draft kept per chain when k > lo). Greedy tokens, metrics and trace equal
    the single-device decode, and equal the same ranks run pipelined."""
    from paper_2509_19368_b200.distributed import StageShard

    config = ppsd.TransformerConfig(8, 512, 8, 8, 64, 1408, 2048, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, 1, exit_stage=k, comm_latency=comm)
    prompt = [int(t) for t in np.random.default_rng(29).integers(0, config.vocab, size=19)]
    full = ppsd.TransformerLM(config, seed=11, deep_scale=0.3, deep_from=k)
    want = ppsd.decode_ppsd(full, cfg, prompt, 48, "greedy", ppsd.RngStream(0), force_reject=force)
    shards = [StageShard(config, cfg, r, world, seed=11, deep_scale=0.3, deep_from=k) for r in range(world)]
    folded = [s.engine.schedule("greedy") == "folded" for s in shards]
    assert any(folded), "no rank folds in this split"
    for sched in ("auto", "pipelined"):
        for s in shards:
            s.engine.set_schedule(sched)
        res = run_loopback(shards, prompt, 48, force_reject=force)
        for toks, m, tr in res:
            assert toks == want[0]
            assert m == want[1]
            assert tr.to_csv() == want[2].to_csv()
        for s, f in zip(shards, folded):
            ran = s.last["schedule"]
            assert ran == ("folded" if f and sched == "auto" else "pipelined"), (sched, ran)
            if ran == "folded":
                # its deferred layers stream once per batch, not once per tick
                # (with k > 1 chains launch k ticks apart: batches of one)
                assert 0 < s.last["deep_batches"] < s.last["ticks"], s.last
                assert s.last["deep_vectors"] >= s.last["deep_batches"], s.last
                if k == 1:
                    assert s.last["deep_vectors"] > s.last["deep_batches"], s.last
