#!/usr/bin/env python
"""Benchmark: greedy PPSD decode tokens/s on Llama-2-shaped models (B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model 7b|13b|70b] [--exit E]

One step = one `decode_ppsd` of 512 new tokens after a 128-token prompt
(prompt 128, decode 512, bs=1). The workload follows
BASELINE.json's configs by GPU count unless --model/--exit override it:

    N=1: Llama-2-7B shape, E=8  (configs[1], single B200, folded schedule)
    N=2: Llama-2-13B shape, E=20 (configs[2], draft | verify over 2 GPUs)
    N=4: Llama-2-70B shape, E=20 (configs[3], one stage per GPU)
    N=8: Llama-2-70B shape, E=10 (configs[3], the paper's PPSD^8)

`value` is committed tokens/s of the decode phase, timed with CUDA events on
the engine stream (prefill excluded, as the paper's decoding-phase numbers;
max over ranks for N > 1); `e2e` times the public `decode_ppsd` call end to
end with host prompt in / host tokens+trace out, prefill included. Weights
(13.5-138 GB) are far larger than the 126 MB L2, so every step streams them
from HBM.

`--impl reference` times the reference algorithm on the host CPU: the
oracle port of specpipe's decode_ppsd machine (oracle/specpipe_port.py)
driving the fp32 CPU decoder (oracle/transformer.py) on the same shape. Each
step decodes a bounded sample (REF_STEP_TOKENS tokens, continuing the same
sequence from step to step) so a `--steps K --warmup W` run ends within a few
minutes; its `value` is tokens/s, the same metric and unit as our arm.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/sec (bs=1) and speedup vs AR at 1/2/4/8 B200; % HBM roofline"
PROMPT_LEN = 128
NEW_TOKENS = 512
EXIT_DEPTH = 8
DEEP_SCALE = 0.08   # residual scale of layers >= E: measured alpha ~0.73 (paper V7B E=8: 0.67-0.81)
SEED = 0
NOMINAL_HBM_GBS = 8000.0   # BASELINE.md §4's denominator (B200 nominal)
REF_STEP_TOKENS = 16       # tokens per reference-arm step (a bounded sample: W+K=25 steps ~ 2.5 min)
EESD_GAMMAS = (5, 10)
# BASELINE.json configs by GPU count: (model, exit depth)
DEFAULTS_BY_N = {1: ("7b", 8), 2: ("13b", 20), 4: ("70b", 20), 8: ("70b", 10)}


def bench_prompt(vocab, n=PROMPT_LEN, seed=SEED):
    """The bench's synthetic prompt: n ids from the seeded `prompt` stream of
    RngStream(derive_seed(seed, "run")) (pipesim.default_prompt's stream)."""
    import paper_2509_19368_b200 as ppsd

    pstream = ppsd.RngStream(ppsd.derive_seed(seed, "run")).split("prompt")
    return [pstream.randbelow(vocab) for _ in range(n)]


def model_config(name):
    import paper_2509_19368_b200 as ppsd

    return {"7b": ppsd.TransformerConfig.llama2_7b, "13b": ppsd.TransformerConfig.llama2_13b,
            "70b": ppsd.TransformerConfig.llama2_70b}[name](max_ctx=1024)


def workload(args, world):
    """(model name, exit depth) for this run: --model/--exit, else BASELINE's config for N."""
    dm, de = DEFAULTS_BY_N.get(world, ("7b", EXIT_DEPTH if world <= 4 else max(1, 32 // world)))
    name = args.model or dm
    exit_depth = args.exit or (de if name == dm else EXIT_DEPTH)
    return name, exit_depth


def tokens_digest(toks):
    """Order-sensitive 40-bit digest of a token list (N=1 and N>1 lines are comparable)."""
    import numpy as np

    return int(np.bitwise_xor.reduce(np.asarray(toks, dtype=np.int64) * 1000003 + np.arange(len(toks)))) & (2**40 - 1)


def workload_label(name, cfg, world):
    where = "1 GPU" if world == 1 else f"{world} GPUs"
    return (f"Llama-2-{name.upper()}-shaped greedy PPSD decode, E={cfg.exit_depth} ({cfg.n_stages} stages on "
            f"{where}), bs=1, prompt {PROMPT_LEN}, {NEW_TOKENS} new tokens")


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "affinity_cores": len(os.sched_getaffinity(0)), "cpu_model": model}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def algorithmic_bytes(trace, config, cfg, n_prompt, last=None):
    """HBM bytes a decode must move.

    Pipelined schedule: stage weights per stage-forward, one tied LM-head pass
    per tick that runs any head, and the KV rows each forward's attention
    reads. Folded schedule: per launched chain its shallow
    stages + the exit-head pass; per deep batch the deep stages + one
    final-head pass (weights counted ONCE per batch: that is the point of
    the batch); KV rows per chain and layer either way."""
    from paper_2509_19368_b200.pipeline import ACTIVATION, CHECK_TOKEN, DRAFT_TOKEN, FINAL_TOKEN

    layer_b = config.layer_bytes()
    kv_b = config.kv_bytes_per_token_layer()
    if last and last.get("schedule") == "folded":
        k = cfg.exit_stage or 1
        shallow = sum(cfg.stage_layers[:k])
        deep = config.n_layers - shallow
        launches = [r.position for r in trace if r.kind == ACTIVATION and r.stage == 1]
        nb, nvec, psum = last["deep_batches"], last["deep_vectors"], last["deep_pos_sum"]
        comb = last.get("comb_heads", 0)  # exit heads that rode in a batch's final-head pass
        weights = len(launches) * shallow * layer_b + nb * deep * layer_b
        heads = (len(launches) + nb - comb) * config.head_bytes()
        kv = (shallow * kv_b * sum(n_prompt + p - 1 for p in launches)
              + deep * kv_b * (psum + nvec * (n_prompt - 1)))
        return weights + heads + kv, dict(schedule="folded", shallow_passes=len(launches),
                                          deep_batches=nb, deep_vectors=nvec, comb_heads=comb, weight_bytes=weights,
                                          head_bytes=heads, kv_bytes=kv)
    head_ticks = set()
    weights = kv = 0
    fwd = 0
    for r in trace:
        if r.kind in (ACTIVATION, FINAL_TOKEN, CHECK_TOKEN):
            nl = cfg.stage_layers[r.stage - 1]
            weights += nl * layer_b
            ctx = n_prompt + r.position - 1  # tokens 0..j attended (j = n_prompt+pos-2)
            kv += nl * ctx * kv_b
            fwd += 1
        if r.kind in (DRAFT_TOKEN, FINAL_TOKEN, CHECK_TOKEN):
            head_ticks.add(r.tick)
    heads = len(head_ticks) * config.head_bytes()
    return weights + heads + kv, dict(schedule="pipelined", stage_forwards=fwd, head_passes=len(head_ticks),
                                      weight_bytes=weights, head_bytes=heads, kv_bytes=kv)


def ar_bytes(config, n_prompt, n_new):
    """Algorithmic bytes of n_new AR tokens: every layer + the final head per
    token, KV rows of the context each token attends."""
    kv = config.n_layers * config.kv_bytes_per_token_layer() * sum(n_prompt + j for j in range(n_new))
    return n_new * (config.n_layers * config.layer_bytes() + config.head_bytes()) + kv


# ---------------------------------------------------------------- ours, N=1 --

def run_ours(args):
    import numpy as np
    import torch

    import paper_2509_19368_b200 as ppsd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PPSD_BENCH_SAME_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        return run_pipelined(args, world, rank, local)

    name, exit_depth = workload(args, 1)
    config = model_config(name)
    cfg = ppsd.PipelineConfig(config.n_layers, exit_depth)
    lm = ppsd.TransformerLM(config, seed=SEED, deep_scale=args.deep_scale, deep_from=exit_depth)
    prompt = bench_prompt(config.vocab)
    eng = ppsd.engine_for(lm, cfg)

    def one_step():
        toks, m, tr = eng.decode(prompt, NEW_TOKENS)
        return toks, m, tr, dict(eng.last)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    steps = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            steps.append(one_step())
        torch.cuda.synchronize()
    dec_ms = [s[3]["decode_ms"] for s in steps]
    toks0, m0, tr0, last0 = steps[0]
    assert all(s[0] == toks0 for s in steps), "decode is not deterministic across steps"
    value = NEW_TOKENS * len(steps) / (sum(dec_ms) / 1e3)
    launches = sum(s[3]["gpu_launches"] for s in steps)

    # the other single-device schedule on the same engine: identical tokens,
    # metrics and trace, its own time
    other = "pipelined" if last0["schedule"] == "folded" else "folded"
    alt = None
    try:
        eng.set_schedule(other)
        alt_ms = []
        for _ in range(max(1, min(3, args.steps))):
            t_, m_, tr_ = eng.decode(prompt, NEW_TOKENS)
            assert t_ == toks0 and m_ == m0 and tr_.to_csv() == tr0.to_csv(), \
                f"{other} schedule differs from {last0['schedule']}"
            alt_ms.append(eng.last["decode_ms"])
        alt_bytes, alt_bd = algorithmic_bytes(tr_, config, cfg, PROMPT_LEN, eng.last)
        alt = {"schedule": other, "tokens_per_s": round(NEW_TOKENS / (np.median(alt_ms) / 1e3), 3),
               "ms_per_step": round(float(np.median(alt_ms)), 3), "gpu_launches": eng.last["gpu_launches"],
               "step_gbs": round(alt_bytes / (np.median(alt_ms) / 1e3) / 1e9, 1), **alt_bd}
    except (ValueError, NotImplementedError, RuntimeError):
        alt = None
    finally:
        eng.set_schedule("auto")

    # end to end through the public API: host prompt -> tokens/trace on host
    rng = ppsd.RngStream(ppsd.derive_seed(SEED, "run"))
    e2e_times = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # one untimed call first: the schedule switch above leaves the engine to
    # rebuild its folded tick graphs on the next decode (one-time setup, like
    # the warm-up steps of the device-timed value)
    ppsd.decode_ppsd(lm, cfg, prompt, NEW_TOKENS, "greedy", rng)
    for _ in range(max(1, args.steps)):
        torch.cuda.synchronize()
        ev0.record()
        t0 = time.perf_counter()
        toks, m, tr = ppsd.decode_ppsd(lm, cfg, prompt, NEW_TOKENS, "greedy", rng)
        t1 = time.perf_counter()
        ev1.record()
        torch.cuda.synchronize()
        e2e_times.append(max(t1 - t0, ev0.elapsed_time(ev1) / 1e3))
        assert toks == toks0
    e2e_val = NEW_TOKENS * len(e2e_times) / sum(e2e_times)

    hbm, peak_kind = peaks()
    # AR baseline on the same engine (same kernels, one chain through all stages)
    ar_ms = []
    for _ in range(max(1, min(3, args.steps))):
        ar = eng.decode_ar(prompt, NEW_TOKENS)
        ar_ms.append(eng.last["decode_ms"])
    assert ar == toks0, "PPSD must equal AR token-for-token"
    ar_tps = NEW_TOKENS / (np.median(ar_ms) / 1e3)
    ar_gbs = ar_bytes(config, PROMPT_LEN, NEW_TOKENS) / (np.median(ar_ms) / 1e3) / 1e9

    # vanilla EESD draft-then-verify on the same engine (pipesim.py:435-551):
    # gamma one-token drafts through the exit layers, one batched verify
    eesd = {}
    for g in EESD_GAMMAS:
        ems = []
        for _ in range(2):
            et, em, _ = eng.decode_eesd(prompt, NEW_TOKENS, g, trace=False)
            ems.append(eng.last["decode_ms"])
        assert et[:NEW_TOKENS] == toks0, "EESD must equal AR"
        a = em.alpha_all_measured
        tps = em.committed_tokens / (np.median(ems) / 1e3)
        eesd[f"gamma{g}"] = {
            "tokens_per_s": round(tps, 3), "alpha_measured": a, "committed": em.committed_tokens,
            "ticks": em.ticks, "tick_speedup": em.speedup_vs_ar, "vs_our_ar": round(tps / ar_tps, 4),
            "eesd_speedup_eq5": ppsd.eesd_speedup(ppsd.SpeedupParams(a, g, config.n_layers, exit_depth))
            if a is not None else None}
    best_eesd = max(v["tokens_per_s"] for v in eesd.values())

    # Roofline of the dominant kernel, timed live with CUDA events on the
    # engine stream (ppsd_probe_gemv: back-to-back launches that walk the
    # stage's layers, so no launch finds its weights in L2). Folded schedule:
    # the gate/up GEMV of a shallow tick (one vector, 180 MB per launch; the
    # largest share of the step in the launch list, profiles/); pipelined: the
    # grouped gate/up launch over all stages. `kernels` lists every layer
    # GEMV as each schedule launches it (tick plan, and the folded deep batch
    # of up to 4 vectors in one weight pass).
    reps = 50
    folded = last0["schedule"] == "folded"
    gu_ms, gu_bytes = eng.probe_gemv(2, 1 if folded else cfg.n_stages, reps)
    achieved = gu_bytes / (gu_ms / 1e3) / 1e9
    kern = {}
    nb = min(cfg.n_stages, 4)
    for wi, nm in enumerate(("qkv", "o", "gate_up", "down")):
        for lab, g in (("tick", 1), (f"tick_x{cfg.n_stages}_stages", cfg.n_stages), (f"batch{nb}", -nb)):
            ms_, b_ = eng.probe_gemv(wi, g, 20)
            kern[f"{nm}_{lab}"] = {"us": round(ms_ * 1e3, 2), "GB/s": round(b_ / (ms_ / 1e3) / 1e9, 1)}
    for lab, (wi, g) in (("head_tick", (4, 1)), (f"head_batch{nb}", (5, -nb))):
        ms_, b_ = eng.probe_gemv(wi, g, 20)
        kern[lab] = {"us": round(ms_ * 1e3, 2), "GB/s": round(b_ / (ms_ / 1e3) / 1e9, 1)}
    step_bytes, breakdown = algorithmic_bytes(tr0, config, cfg, PROMPT_LEN, last0)
    step_gbs = step_bytes / (np.median(dec_ms) / 1e3) / 1e9
    alpha = m0.alpha_all_measured
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemv_gateup_m1_traffic.json" if folded else "gemv_gateup_traffic.json")
    if os.path.exists(tpath) and name == "7b":
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except Exception:
            traffic = None

    toy = toylm_rows() if args.toy_rows and rank == 0 else None
    cpu = cpu_baseline(config, cfg, prompt, args) if args.cpu_budget > 0 else None

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(float(np.mean(dec_ms)), 3),
        "step_tokens": NEW_TOKENS,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: counter-hash random-init weights, seeded random prompt",
        "config": {"workload": workload_label(name, cfg, 1),
                   "model": f"llama2-{name}-shape", "exit_depth": exit_depth, "n_stages": cfg.n_stages,
                   "deep_scale": args.deep_scale, "prompt_len": PROMPT_LEN, "new_tokens": NEW_TOKENS,
                   "kv_dtype": config.kv_dtype, "schedule": last0["schedule"],
                   "parallelism": "pp-stages on 1 GPU (" + last0["schedule"] + " schedule)",
                   "l2": f"inputs larger than L2 ({config.n_layers * config.layer_bytes() / 1e9:.1f} GB "
                         "weights streamed per step)"},
        "e2e": {"value": round(e2e_val, 3), "unit": "tokens/s", "h2d_bytes_per_step": 4 * PROMPT_LEN,
                "d2h_bytes_per_step": 4 * NEW_TOKENS + 24 * len(tr0) + 88,
                "note": "public decode_ppsd call incl. prefill of the 128-token prompt"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "kernel": (f"tcgemv_kernel<gate/up + SwiGLU> (tcgen05), one vector, {gu_bytes / 1e6:.0f} MB per launch"
                                if folded else f"tcgemv_kernel<gate/up>, {cfg.n_stages} stages per launch"),
                     "algorithmic_bytes": gu_bytes, "peak_kind": peak_kind, "avg_ms": round(gu_ms, 4)},
        "kernels": kern,
        "step_roofline": {"achieved": round(step_gbs, 1), "frac": round(step_gbs / hbm, 4),
                          "frac_nominal_8tbs": round(step_gbs / NOMINAL_HBM_GBS, 4),
                          "peak_measured": hbm, "peak_nominal": NOMINAL_HBM_GBS,
                          "bytes_per_step": step_bytes, **breakdown},
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "alpha_measured": alpha, "ticks": m0.ticks, "accepts": m0.accepts, "rejects": m0.rejects,
        "tokens_digest": tokens_digest(toks0),
        "tick_speedup": m0.speedup_vs_ar,
        "ppsd_speedup_eq7": ppsd.ppsd_speedup(alpha, config.n_layers, exit_depth) if alpha is not None else None,
        "ar_tokens_per_s": round(ar_tps, 3), "speedup_vs_our_ar": round(value / ar_tps, 4),
        "ar_step_roofline": {"achieved": round(ar_gbs, 1), "frac": round(ar_gbs / hbm, 4),
                             "frac_nominal_8tbs": round(ar_gbs / NOMINAL_HBM_GBS, 4)},
        "eesd": eesd, "speedup_vs_our_best_eesd": round(value / best_eesd, 4),
        "prefill_ms": round(steps[0][3]["prefill_ms"], 3),
        "other_schedule": alt,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if toy:
        line["toylm_config1"] = toy
    if rank == 0:
        print(json.dumps(line))


# ------------------------------------------------------- ours, N > 1 ranks --

def run_pipelined(args, world, rank, local):
    """N > 1: one pipeline rank per GPU (stages split contiguously). The
    workload is BASELINE's config for N (DEFAULTS_BY_N) unless --model/--exit.
    Transport (PPSD_BENCH_EXCHANGE): `p2p` (default) — NVLink peer stores +
    system-scope flags, a whole tick is one CUDA graph per rank; `nccl` — box
    all-gather between the compute and finish graphs; `host` — gloo through
    host memory (test mode only). Timed on each rank's stream with CUDA
    events; max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2509_19368_b200 as ppsd
    from paper_2509_19368_b200 import distributed as D
    from paper_2509_19368_b200.pipeline import ACTIVATION, CHECK_TOKEN, DRAFT_TOKEN, FINAL_TOKEN

    transport = os.environ.get("PPSD_BENCH_EXCHANGE", "p2p")
    # PPSD_BENCH_SAME_GPU=1: every rank on cuda:0 — exercises this path on one
    # device (a test mode, not a bench). Ranks sharing a device must not use
    # programmatic dependent launch with the p2p spin-waits.
    same_gpu = os.environ.get("PPSD_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
        os.environ["PPSD_PDL"] = "0"
    torch.cuda.set_device(local)
    if transport == "host" or same_gpu:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    reduce_dev = "cpu" if (transport == "host" or same_gpu) else f"cuda:{local}"
    name, exit_depth = workload(args, world)
    config = model_config(name)
    cfg = ppsd.PipelineConfig(config.n_layers, exit_depth)
    shard = D.StageShard(config, cfg, rank, world, seed=SEED, deep_scale=args.deep_scale,
                         deep_from=exit_depth, device=local)
    if transport == "p2p":
        # peer mapping failures (no P2P between the devices) fall back to the
        # NCCL all-gather on every rank, decided collectively
        ok = 1
        try:
            D.p2p_setup_group(shard)
        except Exception as ex:  # noqa: BLE001
            ok = 0
            print(f"rank {rank}: peer-store transport unavailable ({ex}); using nccl", file=sys.stderr)
        flag = torch.tensor([ok], dtype=torch.int32, device=reduce_dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            transport = "nccl"
    if transport == "p2p":

        def decode(prompt):
            return D.decode_ppsd_p2p(shard, prompt, NEW_TOKENS)
    else:
        exchange = D.host_exchange(shard) if transport == "host" else D.nccl_exchange(shard)

        def decode(prompt):
            return D.decode_ppsd_pipelined(shard, prompt, NEW_TOKENS, exchange)
    prompt = bench_prompt(config.vocab)
    for _ in range(args.warmup):
        decode(prompt)
    dist.barrier()
    torch.cuda.synchronize()
    dec, launches, res = [], 0, None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            res = decode(prompt)
            dec.append(shard.last["decode_ms"])
            launches += shard.last["gpu_launches"]
    torch.cuda.synchronize()
    dist.barrier()
    toks, m, tr = res

    # end to end through the per-rank public call (host prompt in, host tokens,
    # metrics and trace out), wall clock, max over ranks
    e2e = []
    for _ in range(max(1, min(3, args.steps))):
        dist.barrier()
        t0 = time.perf_counter()
        out = decode(prompt)
        e2e.append(time.perf_counter() - t0)
        assert out[0] == toks

    # per-rank roofline: this rank's stage weights + KV per stage-forward it
    # ran (ACTIVATION / FINAL / CHECK rows of its stages) + its head passes
    lo, hi = shard.stages
    k = cfg.exit_stage or 1
    rb = 0
    head_ticks = set()
    for r in tr:
        if not lo <= r.stage <= hi:
            continue
        if r.kind in (ACTIVATION, FINAL_TOKEN, CHECK_TOKEN):
            nl = cfg.stage_layers[r.stage - 1]
            rb += nl * (config.layer_bytes() + config.kv_bytes_per_token_layer() * (PROMPT_LEN + r.position - 1))
        if r.kind in (DRAFT_TOKEN, FINAL_TOKEN, CHECK_TOKEN) and (r.stage == k or r.stage == cfg.n_stages):
            head_ticks.add(r.tick)
    rb += len(head_ticks) * config.head_bytes()
    rank_gbs = rb / (float(np.mean(dec)) / 1e3) / 1e9
    hbm, _ = peaks()

    # every rank must hold the same tokens (replicated scheduler)
    digest = tokens_digest(toks)
    agg = torch.tensor([sum(dec), sum(e2e), digest, -digest, -rank_gbs, rank_gbs], dtype=torch.float64,
                       device=reduce_dev)
    dist.all_reduce(agg, op=dist.ReduceOp.MAX)
    total_ms, e2e_s = float(agg[0].item()), float(agg[1].item())
    if int(agg[2].item()) != digest or int(-agg[3].item()) != digest:
        raise RuntimeError("ranks disagree on the decoded tokens")
    value = NEW_TOKENS * args.steps / (total_ms / 1e3)
    if same_gpu or transport == "host":
        print(json.dumps({"rank": rank, "tokens_head": toks[:8], "ticks": m.ticks, "accepts": m.accepts}),
              file=sys.stderr)
    rmin, rmax = -float(agg[4].item()), float(agg[5].item())
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 3),
        "step_tokens": NEW_TOKENS,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: counter-hash random-init weights, seeded random prompt",
        "config": {"workload": workload_label(name, cfg, world),
                   "model": f"llama2-{name}-shape", "exit_depth": exit_depth, "n_stages": cfg.n_stages,
                   "deep_scale": args.deep_scale, "transport": transport,
                   "parallelism": f"pp{world} (stage pipeline, {transport} box exchange per tick)",
                   "l2": "inputs larger than L2 (weights streamed per step)"},
        "e2e": {"value": round(NEW_TOKENS * len(e2e) / e2e_s, 3), "unit": "tokens/s",
                "h2d_bytes_per_step": 4 * PROMPT_LEN, "d2h_bytes_per_step": 4 * NEW_TOKENS + 24 * len(tr) + 88,
                "note": "per-rank public decode call incl. prefill, wall clock, max over ranks"},
        "rank_roofline": {"min_gbs": round(rmin, 1), "max_gbs": round(rmax, 1), "peak": hbm,
                          "min_frac": round(rmin / hbm, 4), "min_frac_nominal_8tbs": round(rmin / NOMINAL_HBM_GBS, 4)},
        "clocks": clk.summary(), "gpu_launches": launches,
        "alpha_measured": m.alpha_all_measured, "ticks": m.ticks, "accepts": m.accepts, "rejects": m.rejects,
        "tokens_digest": digest, "tick_speedup": m.speedup_vs_ar,
        "ppsd_speedup_eq7": ppsd.ppsd_speedup(m.alpha_all_measured, config.n_layers, exit_depth)
        if m.alpha_all_measured is not None else None,
    }
    if rank == 0:
        print(json.dumps(line))
    dist.destroy_process_group()


# ------------------------------------------------------------ CPU reference --

class CpuReference:
    """The reference algorithm on the host: the oracle port of specpipe's
    _ppsd_machine (oracle/specpipe_port.py, pinned to the reference's goldens)
    driving the fp32 numpy decoder (oracle/transformer.py) with every host
    thread. Weights are built once; the prompt is prefilled once (excluded,
    like the GPU value); each step then decodes `n` more tokens of the SAME
    sequence (the oracle's prefix trie makes a repeated prefix free, so steps
    continue rather than restart)."""

    def __init__(self, config, exit_depth, deep_scale, threads=None):
        import numpy as np

        from oracle.transformer import ModelShape, TransformerOracle

        self.threads = threads or os.cpu_count() or 1
        self.config, self.exit_depth = config, exit_depth
        shape = ModelShape(config.n_layers, config.d_model, config.n_heads, config.n_kv_heads,
                           config.head_dim, config.ffn_dim, config.vocab, config.rms_eps, config.rope_theta)
        t0 = time.perf_counter()
        self.lm = TransformerOracle(shape, seed=SEED, deep_scale=deep_scale, deep_from=exit_depth,
                                    dtype=np.float32, max_ctx=config.max_ctx, threads=self.threads,
                                    rope_fp32=True, kv_bf16=config.kv_dtype == "bf16")
        self.init_s = time.perf_counter() - t0
        self.seq = None

    def prefill(self, prompt):
        d = self.lm.empty_digest()
        for t in prompt:
            d = self.lm.extend_digest(d, t)
        self.lm.final_logits(d[0])  # batched prompt forward (excluded from the timing)
        self.seq = list(prompt)

    def step(self, n):
        from oracle import specpipe_port as sp

        t0 = time.perf_counter()
        toks, m, _ = sp.decode_ppsd(self.lm, self.config.n_layers, self.exit_depth, self.seq, n, trace=False)
        dt = time.perf_counter() - t0
        self.seq += toks
        return dt, m

    @staticmethod
    def fits(config):
        """fp32 weights of the shape fit in 70% of host RAM."""
        need = 2 * config.n_layers * config.layer_bytes() + 8 * config.vocab * config.d_model
        try:
            ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        except (ValueError, OSError):
            return True
        return need < 0.7 * ram


def cpu_baseline(config, cfg, prompt, args):
    """Our arm's cpu_baseline: the reference algorithm on this host's cores,
    a bounded sample (1 warm-up + 2 timed steps of REF_STEP_TOKENS tokens)."""
    if not CpuReference.fits(config):
        return None
    ref = CpuReference(config, cfg.exit_depth, args.deep_scale)
    ref.prefill(prompt)
    ref.step(REF_STEP_TOKENS)
    tot, n = 0.0, 0
    for _ in range(2):
        dt, _ = ref.step(REF_STEP_TOKENS)
        tot += dt
        n += REF_STEP_TOKENS
    return {"value": round(n / tot, 4), "unit": "tokens/s", "cores": ref.threads, "kind": "port",
            "sample": f"2 x {REF_STEP_TOKENS} tokens of greedy PPSD (E={cfg.exit_depth}) continuing one "
                      f"sequence after the {PROMPT_LEN}-token prompt (prefill excluded): oracle port of "
                      "pipesim._ppsd_machine + fp32 numpy decoder, same shape and weights",
            "seconds": round(tot, 2), **host_info()}


def toylm_rows():
    """BASELINE config 1 / BASELINE.md §5 items 1 and 3: the reference ToyLM
    decode path (oracle port, bit-exact with specpipe's goldens) on ONE host
    core (affinity = `taskset -c <core>`), next to the same decodes on the GPU."""
    import statistics

    import numpy as np

    import paper_2509_19368_b200 as ppsd
    from oracle import specpipe_port as sp

    lm_seed = sp.derive_seed(0, "lm")
    prompt = sp.default_prompt(16, sp.derive_seed(0, "run"))
    old = os.sched_getaffinity(0)
    core = min(old)
    out = {"config": "ToyLM(32, 16, derive_seed(0,'lm'), beta), PipelineConfig(32, 8), default prompt, 128 tokens",
           "host": {**host_info(), "pinned_core": core}, "cpu_port_1core": {}, "gpu": {}}
    gen = np.random.default_rng(2026)  # pkg/tests/test_acceptance.py:135-145
    cases = []
    for _ in range(200):
        s = int(gen.integers(2**63))
        cases.append((s, [int(x) for x in gen.integers(16, size=8)]))
    os.sched_setaffinity(0, {core})
    try:
        for beta in (1.0, 0.0):
            lm = sp.ToyLMPort(32, 16, lm_seed, beta)
            ts = []
            for _ in range(21):
                t0 = time.perf_counter()
                _, m, _ = sp.decode_ppsd(lm, 32, 8, prompt, 128, trace=False)
                ts.append(time.perf_counter() - t0)
            med = statistics.median(ts)
            out["cpu_port_1core"][f"decode_ppsd_beta{beta:g}"] = {
                "ms": round(med * 1e3, 3), "tokens_per_s": round(128 / med, 1), "ticks": m[1], "accepts": m[2],
                "rejects": m[3]}
        lm = sp.ToyLMPort(32, 16, lm_seed, 1.0)
        ts = []
        for _ in range(21):
            t0 = time.perf_counter()
            sp.decode_autoregressive(lm, prompt, 128)
            ts.append(time.perf_counter() - t0)
        out["cpu_port_1core"]["decode_autoregressive"] = {"ms": round(statistics.median(ts) * 1e3, 3)}
        ts = []
        for s, pr in cases:
            lmc = sp.ToyLMPort(32, 16, s, 1.0)
            t0 = time.perf_counter()
            sp.decode_ppsd(lmc, 32, 8, pr, 128, trace=False)
            ts.append(time.perf_counter() - t0)
        out["cpu_port_1core"]["acceptance200"] = {"median_ms": round(statistics.median(ts) * 1e3, 3),
                                                 "tokens_per_s": round(128 * 200 / sum(ts), 1)}
    finally:
        os.sched_setaffinity(0, old)
    cfg = ppsd.PipelineConfig(32, 8)
    for beta in (1.0, 0.0):
        eng = ppsd.engine_for(ppsd.ToyLM(32, 16, lm_seed, beta), cfg)
        ms = []
        for _ in range(6):
            _, m, _ = eng.decode(prompt, 128, trace=False)
            ms.append(eng.last["decode_ms"])
        med = statistics.median(ms[1:])
        out["gpu"][f"decode_ppsd_beta{beta:g}"] = {"ms": round(med, 3), "tokens_per_s": round(128 / med * 1e3, 1),
                                                   "ticks": m.ticks, "accepts": m.accepts, "rejects": m.rejects}
    tot = 0.0
    for s, pr in cases:
        eng = ppsd.engine_for(ppsd.ToyLM(32, 16, s, 1.0), cfg)
        eng.decode(pr, 128, trace=False)
        tot += eng.last["decode_ms"]
    out["gpu"]["acceptance200"] = {"tokens_per_s": round(128 * 200 / tot * 1e3, 1),
                                   "note": "sum of per-decode CUDA-event times, one engine per model"}
    return out


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2509_19368_b200 as ppsd  # host-side config types only

    name, exit_depth = workload(args, world)
    config = model_config(name)
    cfg = ppsd.PipelineConfig(config.n_layers, exit_depth)
    prompt = bench_prompt(config.vocab)
    if not CpuReference.fits(config):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"fp32 weights of the {name} shape exceed 70% of host RAM"}))
        return
    ref = CpuReference(config, exit_depth, args.deep_scale)
    ref.prefill(prompt)
    room = config.max_ctx - PROMPT_LEN - cfg.n_stages * cfg.hop_period - 8
    step_tokens = max(1, min(REF_STEP_TOKENS, room // max(1, args.warmup + args.steps)))
    for _ in range(args.warmup):
        ref.step(step_tokens)
    times = []
    for _ in range(args.steps):
        dt, _ = ref.step(step_tokens)
        times.append(dt)
    value = step_tokens * len(times) / sum(times)
    sample = (f"{args.steps} timed steps (after {args.warmup} warm-up) of {step_tokens} greedy PPSD tokens "
              f"(E={exit_depth}) continuing one sequence after the {PROMPT_LEN}-token prompt (prefill excluded): "
              "oracle port of pipesim._ppsd_machine + fp32 numpy decoder, same shape and weights as our arm")
    cpu = {"value": round(value, 4), "unit": "tokens/s", "cores": ref.threads, "kind": "port", "sample": sample,
           "weights_init_s": round(ref.init_s, 1), **host_info()}
    line = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * sum(times) / len(times), 3), "step_tokens": step_tokens,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic: counter-hash random-init weights, seeded random prompt",
            "config": {"workload": workload_label(name, cfg, world), "model": f"llama2-{name}-shape",
                       "exit_depth": exit_depth, "n_stages": cfg.n_stages, "deep_scale": args.deep_scale,
                       "prompt_len": PROMPT_LEN, "kv_dtype": config.kv_dtype},
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", choices=["7b", "13b", "70b"], default=None,
                    help="model shape (default: BASELINE's config for the GPU count)")
    ap.add_argument("--exit", type=int, default=None, help="exit depth E (default: BASELINE's for the config)")
    ap.add_argument("--deep-scale", type=float, default=DEEP_SCALE)
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="0 disables the cpu_baseline sample of our arm")
    ap.add_argument("--no-toy-rows", dest="toy_rows", action="store_false",
                    help="skip the ToyLM (config 1) CPU/GPU rows")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
