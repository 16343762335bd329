"""Multi-rank protocol on CPU: world-size 2 and 4 over gloo.

Each process holds a replica of the shipped tick machine (csrc/sched.h, host
build) and computes only its own stages (ToyLM compute from the oracle port,
standing in for the GPU layer kernels); per tick the ranks all-gather one box
each {exit_tok, final_tok, act_slot, activation} exactly like the NCCL path
(ppsd_step_compute -> all_gather -> ppsd_step_finish). Every rank must end
with the reference's tokens, metrics and trace.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden

CASES = [c for c in load_golden("toylm_decode.json")
         if c["max_tokens"] > 0 and c["cfg"].get("comm_latency", 0) == 0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, case_idx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(__file__))
        from hostsched import HostSched
        from oracle import specpipe_port as sp
        from paper_2509_19368_b200.distributed import local_stages, stage_owner

        case = CASES[case_idx]
        cfgd = case["cfg"]
        lm = sp.ToyLMPort(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
        hs = HostSched(cfgd["n_layers"], cfgd["exit_depth"], exit_stage=cfgd.get("exit_stage") or 0,
                       model=1, stop=case["max_tokens"], prompt=case["prompt"], toy_seed=lm.seed)
        S, layers = hs.S, hs.layers
        first = [sum(layers[:i]) for i in range(S)]
        owner = stage_owner(S, world)
        lo, hi = local_stages(owner, rank)
        dig = {}
        M64 = (1 << 64) - 1
        while True:
            ok, work, info = hs.plan()
            if not ok:
                break
            launched, exit_slot, final_slot, k = info[1], info[2], info[3], info[6]
            for st in range(lo, hi + 1):  # this rank's stage compute
                slot = work[st]
                if slot < 0:
                    continue
                if st == 1 and launched:
                    dig[slot] = hs.prefix_digest(hs.n_prompt + hs.chain_pos(slot) - 1)
                a = first[st - 1]
                dig[slot] = lm.advance_digest(dig[slot], a, a + layers[st - 1])
            box = torch.full((6,), -1, dtype=torch.int64)
            if lo <= k <= hi and exit_slot >= 0:
                d = dig[exit_slot]
                fin = lm.advance_digest(d, first[k - 1] + layers[k - 1], case["n_layers"])
                box[0] = sp.first_argmax(lm.exit_logits(fin, d))
            if hi == S and final_slot >= 0:
                box[1] = sp.first_argmax(lm.logits(dig[final_slot]))
            if hi < S and work[hi] >= 0:
                v = dig[work[hi]]
                box[2] = work[hi]
                box[3] = v & 0xFFFFFFFF
                box[4] = v >> 32
            boxes = [torch.empty_like(box) for _ in range(world)]
            dist.all_gather(boxes, box)
            if lo > 1 and work[lo - 1] >= 0:  # unpack the arriving activation
                b = boxes[owner[lo - 1]]
                assert int(b[2]) == work[lo - 1]
                dig[work[lo - 1]] = (int(b[3]) | (int(b[4]) << 32)) & M64
            hs.finish(int(boxes[owner[k]][0]), int(boxes[owner[S]][1]))
        m = hs.metrics()
        q.put((rank, hs.tokens(m[0]), list(m), sp.trace_csv(hs.trace_rows())))
    finally:
        dist.destroy_process_group()


FAST = {("survey_b1", 2), ("deep_exit", 2), ("remainder33", 2), ("eight_stage", 4),
        ("deep_exit3_lat1", 2), ("two_stage", 2), ("vocab1000", 4)}


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case_idx", range(len(CASES)), ids=[c["name"] for c in CASES])
def test_replicated_scheduler_over_gloo(world, case_idx, request):
    case = CASES[case_idx]
    if (case["name"], world) not in FAST and not request.config.getoption("-m") == "slow":
        pytest.skip("covered by the fast subset; run with -m slow for the full grid")
    n_stages = -(-case["cfg"]["n_layers"] // case["cfg"]["exit_depth"])
    if world > n_stages:
        pytest.skip("more ranks than stages")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, case_idx, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, toks, metrics, csv in results:
        assert toks == case["tokens"], rank
        assert metrics == case["metrics"], rank
        assert csv == case["trace_csv"], rank


# ---------------------------------------------------------------------------
# Sampling mode across ranks (ppsd_step_mode): the boxes also carry the exit
# and final distributions of the heads a rank owns, and every rank makes the
# same draft / verify / commit draws from the owners' distributions. Checked
# against the reference's own sampling runs (tests/golden/toylm_sampling.json).

SCASES = [c for c in load_golden("toylm_sampling.json")
          if c.get("kind") is None and c["cfg"].get("comm_latency", 0) == 0]


def _sampling_rank_main(rank, world, port, case_idx, force_reject, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        import numpy as np

        sys.path.insert(0, os.path.dirname(__file__))
        from hostsched import HostSched
        from oracle import specpipe_port as sp
        from paper_2509_19368_b200.distributed import local_stages, stage_owner

        case = SCASES[case_idx]
        cfgd = case["cfg"]
        V = case["vocab"]
        lm = sp.ToyLMPort(case["n_layers"], V, case["lm_seed"], case["beta"])
        hs = HostSched(cfgd["n_layers"], cfgd["exit_depth"], exit_stage=cfgd.get("exit_stage") or 0,
                       model=1, stop=case["max_tokens"], prompt=case["prompt"], toy_seed=lm.seed,
                       force_reject=force_reject)
        rng = sp.Stream(case["rng_seed"])
        s_draft, s_verify, s_commit = rng.split("draft"), rng.split("verify"), rng.split("commit")
        S, layers = hs.S, hs.layers
        first = [sum(layers[:i]) for i in range(S)]
        owner = stage_owner(S, world)
        lo, hi = local_stages(owner, rank)
        dig, pdist = {}, {}
        M64 = (1 << 64) - 1
        while True:
            ok, work, info = hs.plan()
            if not ok:
                break
            launched, exit_slot, final_slot, k = info[1], info[2], info[3], info[6]
            for st in range(lo, hi + 1):
                slot = work[st]
                if slot < 0:
                    continue
                if st == 1 and launched:
                    dig[slot] = hs.prefix_digest(hs.n_prompt + hs.chain_pos(slot) - 1)
                a = first[st - 1]
                dig[slot] = lm.advance_digest(dig[slot], a, a + layers[st - 1])
            hdr = torch.full((3,), -1, dtype=torch.int64)
            dists = torch.zeros(2 * V, dtype=torch.float64)
            if lo <= k <= hi and exit_slot >= 0:
                d = dig[exit_slot]
                fin = lm.advance_digest(d, first[k - 1] + layers[k - 1], case["n_layers"])
                dists[:V] = torch.from_numpy(sp._probs(lm.exit_dist_from_states(sp._State(fin), sp._State(d))))
            if hi == S and final_slot >= 0:
                dists[V:] = torch.from_numpy(sp._probs(lm.dist_from_final_state(sp._State(dig[final_slot]))))
            if hi < S and work[hi] >= 0:
                v = dig[work[hi]]
                hdr[0], hdr[1], hdr[2] = work[hi], v & 0xFFFFFFFF, v >> 32
            hdrs = [torch.empty_like(hdr) for _ in range(world)]
            boxes = [torch.empty_like(dists) for _ in range(world)]
            dist.all_gather(hdrs, hdr)
            dist.all_gather(boxes, dists)
            if lo > 1 and work[lo - 1] >= 0:
                h = hdrs[owner[lo - 1]]
                assert int(h[0]) == work[lo - 1]
                dig[work[lo - 1]] = (int(h[1]) | (int(h[2]) << 32)) & M64
            # replicated draws, verdict first (separate streams)
            final_ok, final_tok = -1, -1
            if final_slot >= 0:
                qd = boxes[owner[S]][V:].numpy()
                pd = pdist[final_slot]
                dtok = hs.chain_tok(final_slot)
                if force_reject:
                    final_ok, final_tok = 0, sp.sample_token(qd, s_commit)
                elif sp.accept_draft(pd[dtok], qd[dtok], s_verify):
                    final_ok, final_tok = 1, dtok
                else:
                    final_ok, final_tok = 0, sp.sample_token(sp.residual(pd, qd), s_commit)
            exit_tok = -1
            if exit_slot >= 0:
                pd = np.array(boxes[owner[k]][:V].numpy())
                pdist[exit_slot] = pd
                exit_tok = sp.sample_token(pd, s_draft)
            hs.finish(exit_tok, final_tok, final_ok)
        m = hs.metrics()
        q.put((rank, hs.tokens(m[0]), list(m), sp.trace_csv(hs.trace_rows())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case_idx", range(len(SCASES)), ids=[c["name"] for c in SCASES])
def test_replicated_sampling_over_gloo(world, case_idx):
    case = SCASES[case_idx]
    n_stages = -(-case["cfg"]["n_layers"] // case["cfg"]["exit_depth"])
    if world > n_stages:
        pytest.skip("more ranks than stages")
    if world == 4 and case["name"] not in ("s_b1", "s_deep_exit"):
        pytest.skip("world 4: two cases keep the CPU suite short")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sampling_rank_main, args=(r, world, port, case_idx, False, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, toks, metrics, csv in results:
        assert toks == case["tokens"], rank
        assert metrics == case["metrics"], rank
        assert csv == case["trace_csv"], rank


def test_replicated_sampling_force_reject_over_gloo():
    """force_reject in sampling mode: every verdict commits a commit-stream
    draw from q (full_model_token, pipesim.py:360-365)."""
    idx = [c["name"] for c in SCASES].index("s_b1")
    case = SCASES[idx]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sampling_rank_main, args=(r, 2, port, idx, True, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0][1] == results[1][1]
    for rank, toks, metrics, csv in results:
        assert metrics == case["force_reject_metrics"], rank
