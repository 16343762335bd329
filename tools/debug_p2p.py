"""Debug driver for the peer-store transport on one GPU: `world` stage-range
engines in one process (world=1: a single engine publishing to itself), each
decoding on its own thread; compares with the single-engine decode."""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("PPSD_PDL", "0")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200.distributed import StageShard, decode_ppsd_p2p, p2p_connect, p2p_prepare  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n_tok = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n_prompt = int(sys.argv[3]) if len(sys.argv) > 3 else 5
CONFIG = dict(n_layers=8, d_model=512, n_heads=8, n_kv_heads=8, head_dim=64, ffn_dim=1408, vocab=2048)
config = ppsd.TransformerConfig(**CONFIG, kv_dtype="bf16", max_ctx=512)
cfg = ppsd.PipelineConfig(8, 2)
prompt = [int(t) for t in np.random.default_rng(7).integers(0, config.vocab, size=n_prompt)]
full = ppsd.TransformerLM(config, seed=5, deep_scale=0.3, deep_from=2)
want = ppsd.decode_ppsd(full, cfg, prompt, n_tok, "greedy", ppsd.RngStream(0))
print("reference", want[0], want[1], flush=True)
shards = [StageShard(config, cfg, r, world, seed=5, deep_scale=0.3, deep_from=2) for r in range(world)]
xbufs = [p2p_prepare(s)[1] for s in shards]
for s in shards:
    p2p_connect(s, local_xbufs=xbufs)
print("connected", flush=True)
res = [None] * world
err = [None] * world


def run(i):
    import time
    time.sleep(float(os.environ.get("DEBUG_DELAY", "0")) * i)
    try:
        print("[py rank %d t=%.3f ms] call" % (i, time.monotonic() * 1e3), file=sys.stderr, flush=True)
        res[i] = decode_ppsd_p2p(shards[i], prompt, n_tok)
        print("[py rank %d t=%.3f ms] back" % (i, time.monotonic() * 1e3), file=sys.stderr, flush=True)
    except Exception as ex:  # noqa: BLE001
        err[i] = ex


ths = [threading.Thread(target=run, args=(i,)) for i in range(world)]
for t in ths:
    t.start()
for t in ths:
    t.join(timeout=120)
for i in range(world):
    print("rank", i, "err", err[i], "res", None if res[i] is None else (res[i][0], res[i][1]), flush=True)
    if res[i] is not None:
        print("  match", res[i][0] == want[0], res[i][1] == want[1], res[i][2].to_csv() == want[2].to_csv())
ref_rows = want[2].to_csv().splitlines()
for i in range(world):
    raw = getattr(shards[i], "last_raw", None)
    if raw is None:
        continue
    print("rank", i, "rc", raw[0], "tokens", raw[1])
    rows = raw[2].to_csv().splitlines()
    for a, (x, y) in enumerate(zip(ref_rows, rows)):
        if x != y:
            print("rank", i, "first trace diff at row", a)
            print("\n".join("  ref " + r for r in ref_rows[max(0, a - 6): a + 4]))
            print("\n".join("  got " + r for r in rows[max(0, a - 6): a + 4]))
            break
try:
    from cuda.bindings import runtime as cudart
except ImportError:  # older cuda-python
    from cuda import cudart
box = 4 + CONFIG["d_model"]
for i in range(world):
    host = np.zeros(world, dtype=np.uint64)
    cudart.cudaMemcpy(host.ctypes.data, xbufs[i] + 2 * world * box * 4, 8 * world,
                      cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    print("buffer of rank", i, "flags", host.tolist())
if os.environ.get("DEBUG_LOG"):
    for i in range(world):
        off = 2 * world * box * 4 + 8 * world
        cnt = np.zeros(1, dtype=np.uint64)
        cudart.cudaMemcpy(cnt.ctypes.data, xbufs[i] + off, 8, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        n = int(min(cnt[0], 500))
        log = np.zeros((n, 8), dtype=np.uint64)
        cudart.cudaMemcpy(log.ctypes.data, xbufs[i] + off + 8, 64 * n, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost)
        t0 = int(log[0, 5]) if n else 0
        print("wait log of rank", i)
        for r in log.tolist():
            print("   e=%d flag0=%d flagL=%d hdr0(slot0)=%d hdr1(slotL)=%d waited=%.1fus xerr=%d rank=%d" % (
                r[0], r[1], r[2], np.int32(np.uint32(r[3])), np.int32(np.uint32(r[4])), r[5] / 1e3, r[6], r[7]))
