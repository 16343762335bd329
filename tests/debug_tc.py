"""Debug helper (not collected): teacher-forced logits of small shapes vs the oracle."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2509_19368_b200 as ppsd  # noqa: E402
from test_gpu_parity import _oracle_for  # noqa: E402

SH = {
    "tiny": dict(n_layers=4, d_model=64, n_heads=4, n_kv_heads=4, head_dim=16, ffn_dim=176, vocab=256),
    "mid_gqa": dict(n_layers=4, d_model=1024, n_heads=16, n_kv_heads=4, head_dim=64, ffn_dim=2816, vocab=4096),
}
for name, sh in SH.items():
    for nl in (1, 2, 4):
        sh2 = dict(sh, n_layers=nl) if nl > 1 else dict(sh, n_layers=2)
        config = ppsd.TransformerConfig(**sh2, kv_dtype="fp32", max_ctx=256)
        lm = ppsd.TransformerLM(config, seed=3, deep_scale=0.5, deep_from=1)
        prompt = [int(t) for t in np.random.default_rng(5).integers(0, config.vocab, size=int(sys.argv[1]) if len(sys.argv) > 1 else 3)]
        eng = ppsd.engine_for(lm, ppsd.PipelineConfig(config.n_layers, 1))
        eng.decode_ar(prompt, 1)
        got = eng.read_logits(1).astype(np.float64)
        orc = _oracle_for(config, 3, 0.5, 1)
        want = orc.logits_for_prefix(prompt)
        print(name, config.n_layers, "max|z|", np.abs(want).max(), "max|dz|", np.abs(got - want).max(),
              "argmax", int(np.argmax(got)), int(np.argmax(want)), flush=True)
