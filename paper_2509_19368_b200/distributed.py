"""Pipeline-parallel PPSD across GPUs: one process (rank) per GPU, each owning a
contiguous range of pipeline stages (BASELINE configs 3-4).

Every rank runs the same device tick machine (the scheduler is replicated and
deterministic), so the only traffic is one fixed-size box per rank per tick:
the activation leaving its last local stage plus the exit / final argmax if it
owns those heads. Boxes are all-gathered with NCCL on the engine's stream
between `ppsd_step_compute` and `ppsd_step_finish` (include/ppsd.h). The
prompt prefill is pipelined over the same exchange.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .decode import Engine, _check_mode
from .models import TransformerConfig, TransformerLM
from .pipeline import EventTrace, PipelineConfig, make_metrics


def stage_owner(n_stages: int, world: int) -> list[int]:
    """Contiguous split of stages 1..S over ranks 0..world-1 (index 0 unused)."""
    if not 1 <= world <= n_stages:
        raise ValueError(f"need 1 <= world ({world}) <= n_stages ({n_stages})")
    return [-1] + [(st - 1) * world // n_stages for st in range(1, n_stages + 1)]


def local_stages(owner: list[int], rank: int) -> tuple[int, int]:
    sts = [st for st in range(1, len(owner)) if owner[st] == rank]
    return sts[0], sts[-1]


class StageShard:
    """The layers, heads and engine of one pipeline rank."""

    def __init__(self, config: TransformerConfig, cfg: PipelineConfig, rank: int, world: int, *,
                 seed: int = 0, deep_scale: float = 1.0, deep_from: int | None = None, device=None,
                 exit_head: str = "norm"):
        import torch

        self.cfg, self.rank, self.world = cfg, rank, world
        self.owner = stage_owner(cfg.n_stages, world)
        lo, hi = local_stages(self.owner, rank)
        first = [sum(cfg.stage_layers[:i]) for i in range(cfg.n_stages)]
        layers = (first[lo - 1], first[hi - 1] + cfg.stage_layers[hi - 1])
        k = cfg.exit_stage
        self.lm = TransformerLM(config, seed=seed, deep_scale=deep_scale, deep_from=deep_from,
                                device=device, layers=layers, need_embed=(lo == 1),
                                need_head=(lo <= k <= hi) or hi == cfg.n_stages,
                                # the exit head's decoder layer lives on the exit stage's rank
                                exit_head=exit_head if lo <= k <= hi else "norm")
        self.engine = Engine(self.lm.model_desc(), self.lm.weights_struct(), cfg,
                             device=self.lm.device.index, stage_range=(lo, hi))
        nbytes, stream = C.c_int64(), C.c_void_p()
        _lib.check(_lib.lib().ppsd_exchange_info(self.engine.h, C.byref(nbytes), C.byref(stream)),
                   "exchange_info")
        self.stream_ptr = stream.value
        self.greedy_words = nbytes.value // 4
        self._boxes(self.greedy_words)
        self.stages = (lo, hi)

    def _boxes(self, words: int):
        import torch

        if getattr(self, "outbox", None) is None or self.outbox.numel() != words:
            self.outbox = torch.zeros(words, dtype=torch.float32, device=self.lm.device)
            self.inbox = torch.zeros(self.world, words, dtype=torch.float32, device=self.lm.device)

    def torch_stream(self):
        import torch

        return torch.cuda.ExternalStream(self.stream_ptr, device=self.lm.device)

    # -- the per-rank protocol ------------------------------------------
    def begin(self, prompt, max_tokens: int, force_reject: bool = False, mode: str = "greedy",
              rng=None) -> int:
        """Sampling (pipesim.py:412-414): boxes also carry the exit / final
        logits and every rank makes the same draws (include/ppsd.h
        ppsd_step_mode); rng is the decode's RngStream."""
        _check_mode(mode)
        L = _lib.lib()
        greedy = mode == "greedy"
        seed = 0 if rng is None else rng.seed
        _lib.check(L.ppsd_step_mode(self.engine.h, int(greedy), seed & ((1 << 64) - 1)), "step_mode")
        self._boxes(self.greedy_words + (0 if greedy else 2 * self.lm.vocab))
        p = (C.c_int32 * len(prompt))(*[int(t) for t in prompt])
        own = (C.c_int32 * len(self.owner))(*self.owner)
        _lib.check(L.ppsd_step_begin(self.engine.h, p, len(prompt), max_tokens, int(bool(force_reject)),
                                     own, self.world, self.rank, C.c_void_p(self.outbox.data_ptr()),
                                     C.c_void_p(self.inbox.data_ptr())), "step_begin")
        n = C.c_int32()
        _lib.check(L.ppsd_prefill_steps(self.engine.h, C.byref(n)), "prefill_steps")
        self.max_tokens = max_tokens
        return n.value

    def prefill_compute(self):
        _lib.check(_lib.lib().ppsd_prefill_compute(self.engine.h), "prefill_compute")

    def compute(self):
        _lib.check(_lib.lib().ppsd_step_compute(self.engine.h), "step_compute")

    def finish(self):
        _lib.check(_lib.lib().ppsd_step_finish(self.engine.h), "step_finish")

    def poll(self):
        done, committed, ticks = C.c_int32(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().ppsd_step_poll(self.engine.h, C.byref(done), C.byref(committed),
                                             C.byref(ticks)), "step_poll")
        return bool(done.value), committed.value, ticks.value

    def end(self):
        L = _lib.lib()
        out = np.zeros(self.max_tokens, dtype=np.int32)
        m = _lib.Metrics()
        cap = self.engine._trace_cap(self.max_tokens)
        rows = np.zeros((cap, 6), dtype=np.int32)
        n = C.c_int64()
        _lib.check(L.ppsd_step_end(self.engine.h, out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(m),
                                   rows.ctypes.data_as(C.POINTER(_lib.TraceRowC)), cap, C.byref(n)),
                   "step_end")
        metrics = make_metrics(m.committed_tokens, m.ticks, m.accepts, m.rejects, m.accepts + m.rejects,
                               self.cfg.ar_ticks_per_token)
        self.last = dict(decode_ms=m.decode_ms, prefill_ms=m.prefill_ms, gpu_launches=m.gpu_launches,
                         ticks=m.ticks, schedule=_lib.schedule_name(m.schedule), deep_batches=m.deep_batches,
                         deep_vectors=m.deep_vectors)
        return out.tolist(), metrics, EventTrace.from_array(rows[: n.value])


def nccl_exchange(shard: StageShard, group=None):
    """all_gather of the per-rank boxes on the engine stream (NVLink / NVSwitch)."""
    import torch
    import torch.distributed as dist

    stream = shard.torch_stream()

    def exchange():
        with torch.cuda.stream(stream):
            dist.all_gather_into_tensor(shard.inbox.view(-1), shard.outbox, group=group)

    return exchange


def decode_ppsd_pipelined(shard: StageShard, prompt, max_tokens: int, exchange=None, *,
                          force_reject: bool = False, mode: str = "greedy", rng=None):
    """PPSD decode with this rank's stages (greedy, or sampling with the
    decode's RngStream); every rank calls it with the same arguments. Returns
    (tokens, RunMetrics, EventTrace), identical on all ranks and identical to
    the single-GPU `decode_ppsd`."""
    exchange = exchange or nccl_exchange(shard)
    steps = shard.begin(prompt, max_tokens, force_reject, mode=mode, rng=rng)
    for _ in range(steps):
        shard.prefill_compute()
        exchange()
    committed = 0
    while True:
        # every rank sees the same replicated state, so every rank launches
        # the same number of ticks and the collectives stay matched
        for _ in range(max(1, max_tokens - committed)):
            shard.compute()
            exchange()
            shard.finish()
        done, committed, _ = shard.poll()
        if done:
            break
    return shard.end()


def host_exchange(shard: StageShard, group=None):
    """The same box all-gather through host memory over a gloo group. Slow;
    only for exercising the multi-rank path when the ranks share one GPU
    (NCCL refuses two ranks on one device)."""
    import torch
    import torch.distributed as dist

    world = shard.world

    def exchange():
        torch.cuda.synchronize(shard.lm.device)
        out = shard.outbox.cpu()
        boxes = [torch.empty_like(out) for _ in range(world)]
        dist.all_gather(boxes, out, group=group)
        shard.inbox.copy_(torch.stack(boxes))
        torch.cuda.synchronize(shard.lm.device)

    return exchange


# ---------------------------------------------------------------------------
# NVLink peer-store transport: boxes are stored by the pack kernel directly
# into every rank's exchange buffer (CUDA IPC), flags released at system
# scope; a whole tick is one graph and the host only launches ticks.


def p2p_prepare(shard: StageShard) -> tuple[bytes, int]:
    """Allocate this rank's exchange buffer; returns (IPC handle bytes, device pointer)."""
    handle = (C.c_char * 64)()
    xbuf = C.c_void_p()
    _lib.check(_lib.lib().ppsd_p2p_prepare(shard.engine.h, shard.world, handle, C.byref(xbuf)), "p2p_prepare")
    return bytes(handle), xbuf.value


def p2p_connect(shard: StageShard, handles: list[bytes] | None = None, local_xbufs: list[int] | None = None):
    """Map the peers' exchange buffers: IPC handles (one process per GPU) or raw
    device pointers (engines sharing one process)."""
    own = (C.c_int32 * len(shard.owner))(*shard.owner)
    if local_xbufs is not None:
        arr = (C.c_void_p * shard.world)(*local_xbufs)
        rc = _lib.lib().ppsd_p2p_connect(shard.engine.h, shard.rank, None, arr, own)
    else:
        blob = C.create_string_buffer(b"".join(handles), 64 * shard.world)
        rc = _lib.lib().ppsd_p2p_connect(shard.engine.h, shard.rank, blob, None, own)
    _lib.check(rc, "p2p_connect")
    shard.transport = "p2p"


def p2p_setup_group(shard: StageShard, group=None):
    """Exchange IPC handles over torch.distributed (any backend) and connect."""
    import torch.distributed as dist

    handle, _ = p2p_prepare(shard)
    handles = [None] * shard.world
    dist.all_gather_object(handles, handle, group=group)
    p2p_connect(shard, handles=handles)


def decode_ppsd_p2p(shard: StageShard, prompt, max_tokens: int, *, force_reject: bool = False,
                    mode: str = "greedy", rng=None):
    """The pipelined decode over the peer-store transport (after p2p_connect),
    greedy or sampling (the boxes then carry the owners' logits); every rank
    calls it with the same arguments."""
    _check_mode(mode)
    L = _lib.lib()
    seed = 0 if rng is None else rng.seed
    _lib.check(L.ppsd_step_mode(shard.engine.h, int(mode == "greedy"), seed & ((1 << 64) - 1)), "step_mode")
    p = (C.c_int32 * len(prompt))(*[int(t) for t in prompt])
    out = np.zeros(max_tokens, dtype=np.int32)
    m = _lib.Metrics()
    cap = shard.engine._trace_cap(max_tokens)
    rows = np.zeros((cap, 6), dtype=np.int32)
    n = C.c_int64()
    rc = L.ppsd_p2p_decode(shard.engine.h, p, len(prompt), max_tokens, int(bool(force_reject)),
                           out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(m),
                           rows.ctypes.data_as(C.POINTER(_lib.TraceRowC)), cap, C.byref(n))
    shard.last_raw = (rc, out.tolist(), EventTrace.from_array(rows[: n.value]))
    _lib.check(rc, "p2p_decode")
    metrics = make_metrics(m.committed_tokens, m.ticks, m.accepts, m.rejects, m.accepts + m.rejects,
                           shard.cfg.ar_ticks_per_token)
    shard.last = dict(decode_ms=m.decode_ms, prefill_ms=m.prefill_ms, gpu_launches=m.gpu_launches, ticks=m.ticks,
                      schedule=_lib.schedule_name(m.schedule), deep_batches=m.deep_batches,
                      deep_vectors=m.deep_vectors)
    return out.tolist(), metrics, EventTrace.from_array(rows[: n.value])
