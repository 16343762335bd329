"""harness.run / sweep on the GPU tick machine vs the reference harness
(tests/golden/harness.json): results rows with the analytic column, the
measured ToyLM acceptance rates (ppsd_toy_alignment) and traces."""

import io

import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

GOLD = {c["kind"]: c for c in load_golden("harness.json")}


@pytest.mark.parametrize("case", GOLD["runs"]["cases"],
                         ids=lambda c: f"{c['config']['regime']}-{c['config'].get('oracle')}-{c['config']['seed']}")
def test_run_rows_match_reference(case):
    from paper_2509_19368_b200 import harness as H

    res = H.run(H.ExperimentConfig(**case["config"]), want_trace=True)
    assert H.result_row(res) == case["row"]
    assert res.measured_alpha == case["measured_alpha"]
    assert res.trace.to_csv() == case["trace_csv"]


@pytest.mark.parametrize("case", GOLD["align"]["cases"], ids=lambda c: f"{c['lm_seed']}-{c['exit_depth']}")
def test_toylm_alignment_matches_reference(case):
    import paper_2509_19368_b200 as ppsd

    lm = ppsd.ToyLM(case["n_layers"], case["vocab"], case["lm_seed"], case["beta"])
    assert lm.empirical_alpha(case["exit_depth"], 200) == case["empirical_alpha"]
    assert lm.greedy_agreement(case["exit_depth"], 200) == case["greedy_agreement"]
    assert lm.empirical_alpha(case["exit_depth"], 37, eval_seed=12345) == case["empirical_alpha_seeded"]


def test_sweep_csv_matches_reference():
    from paper_2509_19368_b200 import harness as H

    spec = H.SweepSpec.from_dict(dict(base=dict(regime="ppsd", n_layers=32, exit_depth=8, horizon=48,
                                                oracle="bernoulli", alpha=0.5, seed=3),
                                      axes={"alpha": [0.3, 0.9], "exit_depth": [4, 8]}))
    buf = io.StringIO()
    H.write_results_csv(H.sweep(spec), buf)
    assert buf.getvalue() == GOLD["sweep"]["csv"]
