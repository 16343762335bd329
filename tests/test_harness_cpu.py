"""Harness (paper_2509_19368_b200.harness) host logic vs the reference's
harness (tests/golden/harness.json, made by tests/golden/make_golden.py):
config validation (field + message), the analytic report, CSV formatting."""

import pytest

from conftest import load_golden
from paper_2509_19368_b200 import harness as H

GOLD = {c["kind"]: c for c in load_golden("harness.json")}


@pytest.mark.parametrize("case", GOLD["bad"]["cases"], ids=lambda c: str(c.get("field")))
def test_config_validation_matches_reference(case):
    if case["error"] is None:
        H.ExperimentConfig(**case["config"])
        return
    with pytest.raises(H.ConfigError) as exc:
        H.ExperimentConfig(**case["config"])
    assert exc.value.field == case["field"]
    assert str(exc.value) == case["error"]


@pytest.mark.parametrize("case", GOLD["report"]["cases"], ids=lambda c: str(c["args"]))
def test_analytic_report_matches_reference(case):
    assert H.analytic_report(*case["args"]) == case["text"]


def test_config_roundtrip(tmp_path):
    for case in GOLD["runs"]["cases"]:
        cfg = H.ExperimentConfig(**case["config"])
        p = tmp_path / "c.json"
        cfg.to_json(p)
        assert H.ExperimentConfig.from_json(p) == cfg
    with pytest.raises(H.ConfigError):
        H.ExperimentConfig.from_dict(dict(regime="ppsd", n_layers=4))
    with pytest.raises(H.ConfigError):
        H.SweepSpec.from_dict(dict(base=dict(regime="autoregressive", n_layers=4, exit_depth=2, horizon=3),
                                   axes={"out": ["x"]}))


def test_results_csv_format():
    from paper_2509_19368_b200.pipeline import RunMetrics

    cfg = H.ExperimentConfig(regime="ppsd", n_layers=32, exit_depth=8, horizon=10, oracle="toylm-greedy", beta=1.0)
    res = H.RunResult(cfg, RunMetrics(10, 23, 6, 4, 0.6, 10 / 23, 40 / 23), 2.0 / 3.0, 0.5, None)
    assert H.result_row(res) == "ppsd,32,8,,,1,0,10,10,23,6,4,0.6,0.4347826087,1.739130435,0.6666666667"
