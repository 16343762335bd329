"""tcgen05 prefill vs batched-GEMV prefill: final logits after a prompt, and
chunk-size invariance of the tcgen05 path (chunk 16 vs 1 must be bit-equal)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_19368_b200 as ppsd  # noqa: E402
from paper_2509_19368_b200.decode import Engine  # noqa: E402

SHAPES = {
    "small": dict(n_layers=4, d_model=512, n_heads=8, n_kv_heads=8, head_dim=64, ffn_dim=1408, vocab=2048),
    "mid_gqa": dict(n_layers=4, d_model=1024, n_heads=16, n_kv_heads=4, head_dim=64, ffn_dim=2816, vocab=4096),
    "l7b_2layer": dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=32, head_dim=128, ffn_dim=11008,
                       vocab=32000),
}


def logits(lm, cfg, prompt, umma, chunk):
    os.environ["PPSD_UMMA"] = str(umma)
    os.environ["PPSD_PREFILL_CHUNK"] = str(chunk)
    eng = Engine(lm.model_desc(), lm.weights_struct(), cfg, device=lm.device.index)
    toks = eng.decode_ar(prompt, 4)
    z = eng.read_logits(1).copy()
    pre = eng.last.get("prefill_ms")
    return z, toks, pre


for name in sys.argv[1:] or list(SHAPES):
    for kv in ("fp32", "bf16"):
        config = ppsd.TransformerConfig(**SHAPES[name], kv_dtype=kv, max_ctx=256)
        lm = ppsd.TransformerLM(config, seed=3, deep_scale=0.5, deep_from=1)
        prompt = [int(t) for t in np.random.default_rng(5).integers(0, config.vocab, size=70)]
        cfg = ppsd.PipelineConfig(config.n_layers, 1)
        zg, tg, pg = logits(lm, cfg, prompt, 0, 16)
        zu, tu, pu = logits(lm, cfg, prompt, 1, 16)
        z1, t1, p1 = logits(lm, cfg, prompt, 1, 1)
        scale = float(np.abs(zg).max())
        print(f"{name}/{kv}: max|z| {scale:.3f}  |umma-gemv| {np.abs(zu - zg).max():.3e}  "
              f"chunk16==chunk1 {bool(np.array_equal(zu, z1))} (max diff {np.abs(zu - z1).max():.3e})  "
              f"tokens gemv {tg} umma {tu} chunk1 {t1}  prefill ms gemv {pg} umma {pu} umma-chunk1 {p1}",
              flush=True)
