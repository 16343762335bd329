"""Debug helper (not collected): tiny transformer golden case, AR / pipelined / folded tokens."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2509_19368_b200 as ppsd  # noqa: E402

case = json.load(open("tests/golden/transformer.json"))["cases"][0]
lm = ppsd.TransformerLM(ppsd.TransformerConfig.tiny(), seed=case["seed"], deep_scale=case["deep_scale"],
                        deep_from=case["deep_from"])
print("golden  ", case["tokens"][:12])
ar = ppsd.decode_autoregressive(lm, case["prompt"], case["max_tokens"], "greedy", ppsd.RngStream(0))
print("AR      ", ar[:12])
for sched in ("pipelined", "folded"):
    lm.schedule = sched
    toks, m, tr = ppsd.decode_ppsd(lm, ppsd.PipelineConfig(**case["cfg"]), case["prompt"], case["max_tokens"],
                                   "greedy", ppsd.RngStream(0))
    print(f"{sched:9s}", toks[:12], m.accepts, m.rejects)
sys.path.insert(0, "tests")
from test_gpu_parity import _oracle_for  # noqa: E402
c = ppsd.TransformerConfig.tiny()
orc = _oracle_for(c, case["seed"], case["deep_scale"], case["deep_from"])
lm.schedule = "auto"
eng = ppsd.Engine(lm.model_desc(), lm.weights_struct(), ppsd.PipelineConfig(c.n_layers, 8),
                  device=lm.device.index)
for n in (1, 2, 3, 5):
    toks = eng.decode_ar(case["prompt"], n)
    got = eng.read_logits(1).astype(np.float64)
    want = orc.logits_for_prefix(case["prompt"] + list(toks[:-1]))
    print(n, toks, "max|dz|", np.abs(got - want).max(), "argmax", int(np.argmax(got)), int(np.argmax(want)))
