"""The reference-side binding printed in INTEGRATION.md ("The binding a
maintainer would add", pkg/src/specpipe/_b200.py) executed verbatim against
this repo's libppsd.so, with the reference's pipesim types replaced by this
package's drop-in mirrors (pipeline.py): CPU — its ctypes structs match the
library's layouts (sizes and field offsets of _lib, which test_library_cpu
pins to include/ppsd.h); GPU — decode_ppsd_b200 reproduces the reference's
ToyLM goldens (tokens, RunMetrics, trace CSV)."""
import ctypes as C
import json
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _binding():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as fh:
        text = fh.read()
    sec = text.index("## The binding a maintainer would add")
    code = re.search(r"```python\n(.*?)```", text[sec:], re.S).group(1)
    code = code.replace("from .pipesim import RunMetrics, EventTrace, StageMessage",
                        "from paper_2509_19368_b200.pipeline import RunMetrics, EventTrace, StageMessage")
    lib = os.path.join(ROOT, "paper_2509_19368_b200", "libppsd.so")
    if not os.path.exists(lib):
        pytest.skip("libppsd.so not built")
    code = code.replace('C.CDLL("libppsd.so")', f"C.CDLL({lib!r})")
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)  # noqa: S102
    return ns


def test_binding_structs_match_library_layouts():
    from paper_2509_19368_b200 import _lib

    ns = _binding()
    for mine, theirs in ((ns["_Model"], _lib.ModelDesc), (ns["_Pipe"], _lib.PipelineDesc),
                         (ns["_Metrics"], _lib.Metrics), (ns["_Row"], _lib.TraceRowC)):
        assert C.sizeof(mine) == C.sizeof(theirs), mine.__name__
        assert [f[0] for f in mine._fields_] == [f[0] for f in theirs._fields_], mine.__name__
        for (name, _), (name2, _) in zip(mine._fields_, theirs._fields_):
            assert getattr(mine, name).offset == getattr(theirs, name2).offset, (mine.__name__, name, name2)


def _golden(name):
    with open(os.path.join(ROOT, "tests", "golden", name)) as fh:
        return json.load(fh)["cases"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", _golden("toylm_decode.json"), ids=lambda c: c["name"])
def test_binding_decode_matches_reference_goldens(case):
    import paper_2509_19368_b200 as ppsd

    ns = _binding()
    lm = ppsd.ToyLM(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    c = case["cfg"]
    cfg = ppsd.PipelineConfig(c["n_layers"], c["exit_depth"], c.get("exit_stage"), c.get("comm_latency", 0))
    toks, m, tr = ns["decode_ppsd_b200"](lm, cfg, case["prompt"], case["max_tokens"], "greedy",
                                         ppsd.RngStream(case["rng_seed"]))
    assert toks == case["tokens"]
    assert [m.committed_tokens, m.ticks, m.accepts, m.rejects, m.alpha_all_measured, m.throughput,
            m.speedup_vs_ar] == case["metrics"]
    assert tr.to_csv() == case["trace_csv"]
