"""The NVLink peer-store transport on ONE GPU.

(1) engines sharing a process: 2 and 4 stage-range engines, peers given as
raw device pointers, each driven by its own host thread (ctypes drops the
GIL), the whole tick — boxes stored into the peers' buffers, system-scope
release/acquire flags, replicated scheduler — running on the device;
(2) two processes on the same GPU exchanging CUDA IPC handles over gloo,
the exact multi-GPU code path. Tokens, metrics and trace must equal the
single-engine decode."""

import os
import socket
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ppsd = pytest.importorskip("paper_2509_19368_b200")

CONFIG = dict(n_layers=8, d_model=512, n_heads=8, n_kv_heads=8, head_dim=64, ffn_dim=1408, vocab=2048)


def _reference(e, prompt, n):
    config = ppsd.TransformerConfig(**CONFIG, kv_dtype="bf16", max_ctx=512)
    full = ppsd.TransformerLM(config, seed=5, deep_scale=0.3, deep_from=e)
    return ppsd.decode_ppsd(full, ppsd.PipelineConfig(8, e), prompt, n, "greedy", ppsd.RngStream(0))


@pytest.mark.parametrize("world,e", [(2, 2), (4, 2), (2, 3)])
def test_p2p_threads_equal_single_gpu(world, e, monkeypatch):
    # Engines sharing ONE GPU must not use programmatic dependent launch: a
    # rank's next GEMV would be scheduled early onto every SM, parked behind
    # its own flag-waiting scheduler kernel, and starve the peer engine whose
    # publish it waits for. On separate GPUs (the real topology) each rank has
    # its own SMs and PDL stays on (the IPC test below keeps it on).
    monkeypatch.setenv("PPSD_PDL", "0")
    from paper_2509_19368_b200.distributed import StageShard, decode_ppsd_p2p, p2p_connect, p2p_prepare

    config = ppsd.TransformerConfig(**CONFIG, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, e)
    if world > cfg.n_stages:
        pytest.skip("more ranks than stages")
    prompt = [int(t) for t in np.random.default_rng(7).integers(0, config.vocab, size=21)]
    want_t, want_m, want_tr = _reference(e, prompt, 80)
    shards = [StageShard(config, cfg, r, world, seed=5, deep_scale=0.3, deep_from=e) for r in range(world)]
    xbufs = [p2p_prepare(s)[1] for s in shards]
    for s in shards:
        p2p_connect(s, local_xbufs=xbufs)
    for _ in range(2):  # twice: exchange numbers keep increasing across calls
        results = [None] * world

        def run(i):
            results[i] = decode_ppsd_p2p(shards[i], prompt, 80)

        threads = [threading.Thread(target=run, args=(i,)) for i in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert not any(t.is_alive() for t in threads), "p2p decode hung"
        for toks, m, tr in results:
            assert toks == want_t
            assert m == want_m
            assert tr.to_csv() == want_tr.to_csv()



@pytest.mark.parametrize("world,k", [(2, 1), (4, 3)])
def test_p2p_threads_decoder_layer_exit_head(world, k, monkeypatch):
    """The Table-1 exit head over the peer-store transport: the exit rank runs
    the head layer inside its tick graph (prefill included)."""
    monkeypatch.setenv("PPSD_PDL", "0")
    from paper_2509_19368_b200.distributed import StageShard, decode_ppsd_p2p, p2p_connect, p2p_prepare

    config = ppsd.TransformerConfig(**CONFIG, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, 2, exit_stage=k)
    prompt = [int(t) for t in np.random.default_rng(9).integers(0, config.vocab, size=17)]
    full = ppsd.TransformerLM(config, seed=4, deep_scale=0.3, deep_from=2, exit_head="layer")
    want_t, want_m, want_tr = ppsd.decode_ppsd(full, cfg, prompt, 48, "greedy", ppsd.RngStream(0))
    shards = [StageShard(config, cfg, r, world, seed=4, deep_scale=0.3, deep_from=2, exit_head="layer")
              for r in range(world)]
    xbufs = [p2p_prepare(s)[1] for s in shards]
    for s in shards:
        p2p_connect(s, local_xbufs=xbufs)
    results = [None] * world

    def run(i):
        results[i] = decode_ppsd_p2p(shards[i], prompt, 48)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "p2p decode hung"
    for toks, m, tr in results:
        assert toks == want_t
        assert m == want_m
        assert tr.to_csv() == want_tr.to_csv()


def test_p2p_threads_sampling(monkeypatch):
    """Sampling over the peer-store transport, then greedy again on the same
    connected engines (the exchange numbers keep increasing across calls)."""
    monkeypatch.setenv("PPSD_PDL", "0")
    from paper_2509_19368_b200.distributed import StageShard, decode_ppsd_p2p, p2p_connect, p2p_prepare

    config = ppsd.TransformerConfig(**CONFIG, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, 2)
    prompt = [int(t) for t in np.random.default_rng(13).integers(0, config.vocab, size=15)]
    full = ppsd.TransformerLM(config, seed=5, deep_scale=0.3, deep_from=2)
    shards = [StageShard(config, cfg, r, 2, seed=5, deep_scale=0.3, deep_from=2) for r in range(2)]
    xbufs = [p2p_prepare(s)[1] for s in shards]
    for s in shards:
        p2p_connect(s, local_xbufs=xbufs)
    for mode, seed in (("sampling", 17), ("greedy", 0), ("sampling", 3)):
        want_t, want_m, want_tr = ppsd.decode_ppsd(full, cfg, prompt, 40, mode, ppsd.RngStream(seed))
        results = [None] * 2

        def run(i):
            results[i] = decode_ppsd_p2p(shards[i], prompt, 40, mode=mode, rng=ppsd.RngStream(seed))

        threads = [threading.Thread(target=run, args=(i,)) for i in range(2)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert not any(t.is_alive() for t in threads), "p2p decode hung"
        for toks, m, tr in results:
            assert toks == want_t, mode
            assert m == want_m, mode
            assert tr.to_csv() == want_tr.to_csv(), mode

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _ipc_rank(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2509_19368_b200 as pp
        from paper_2509_19368_b200.distributed import StageShard, decode_ppsd_p2p, p2p_setup_group

        config = pp.TransformerConfig(**CONFIG, kv_dtype="bf16", max_ctx=512)
        shard = StageShard(config, pp.PipelineConfig(8, 2), rank, world, seed=5, deep_scale=0.3, deep_from=2)
        p2p_setup_group(shard)
        dist.barrier()
        prompt = [int(t) for t in np.random.default_rng(7).integers(0, config.vocab, size=21)]
        toks, m, tr = decode_ppsd_p2p(shard, prompt, 48)
        q.put((rank, toks, tuple(m.__dict__.values()), tr.to_csv()))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_p2p_two_processes_ipc():
    import torch.multiprocessing as mp

    prompt = [int(t) for t in np.random.default_rng(7).integers(0, CONFIG["vocab"], size=21)]
    want_t, want_m, want_tr = _reference(2, prompt, 48)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, toks, m, csv in res:
        assert toks == want_t, rank
        assert m == tuple(want_m.__dict__.values()), rank
        assert csv == want_tr.to_csv(), rank


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_threads_rank_fold(world, monkeypatch):
    """Per-rank fold over the peer-store transport: 8 one-layer stages."""
    monkeypatch.setenv("PPSD_PDL", "0")
    from paper_2509_19368_b200.distributed import StageShard, decode_ppsd_p2p, p2p_connect, p2p_prepare

    config = ppsd.TransformerConfig(**CONFIG, kv_dtype="bf16", max_ctx=512)
    cfg = ppsd.PipelineConfig(8, 1)
    prompt = [int(t) for t in np.random.default_rng(31).integers(0, config.vocab, size=17)]
    full = ppsd.TransformerLM(config, seed=5, deep_scale=0.3, deep_from=1)
    want_t, want_m, want_tr = ppsd.decode_ppsd(full, cfg, prompt, 64, "greedy", ppsd.RngStream(0))
    shards = [StageShard(config, cfg, r, world, seed=5, deep_scale=0.3, deep_from=1) for r in range(world)]
    assert any(s.engine.schedule("greedy") == "folded" for s in shards)
    xbufs = [p2p_prepare(s)[1] for s in shards]
    for s in shards:
        p2p_connect(s, local_xbufs=xbufs)
    results = [None] * world

    def run(i):
        results[i] = decode_ppsd_p2p(shards[i], prompt, 64)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "p2p decode hung"
    for toks, m, tr in results:
        assert toks == want_t
        assert m == want_m
        assert tr.to_csv() == want_tr.to_csv()
    assert any(s.last["schedule"] == "folded" and 0 < s.last["deep_batches"] < s.last["ticks"] for s in shards)
