"""bench.py's host-side contract on CPU: the workload per GPU count is
BASELINE.json's (configs 2-4), the token digest is order-sensitive and equal
for equal lists (N=1 vs N>1 lines compare through it), and the per-unit
algorithmic bytes are SURVEY.md §8(a6)'s (404.8 MB per 7B layer, 634 MB
13B, 1.71 GB 70B)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _args(model=None, exit_depth=None):
    return argparse.Namespace(model=model, exit=exit_depth)


def test_workload_per_gpu_count_is_baselines():
    assert bench.workload(_args(), 1) == ("7b", 8)
    assert bench.workload(_args(), 2) == ("13b", 20)
    assert bench.workload(_args(), 4) == ("70b", 20)
    assert bench.workload(_args(), 8) == ("70b", 10)
    assert bench.workload(_args("13b", 10), 1) == ("13b", 10)
    with open(os.path.join(ROOT, "BASELINE.json")) as fh:
        base = json.load(fh)
    assert "tok" in json.dumps(base).lower()


def test_tokens_digest():
    a = [5, 1, 9, 9, 2]
    assert bench.tokens_digest(a) == bench.tokens_digest(list(a))
    assert bench.tokens_digest(a) != bench.tokens_digest(a[::-1])
    assert bench.tokens_digest(a) != bench.tokens_digest(a[:-1])
    assert 0 <= bench.tokens_digest(a) < 2**40


def test_layer_bytes_match_survey():
    mb = {name: bench.model_config(name).layer_bytes() / 1e6 for name in ("7b", "13b", "70b")}
    assert abs(mb["7b"] - 404.8) < 0.1
    assert abs(mb["13b"] - 634.0) < 1.0
    assert abs(mb["70b"] - 1711.0) < 2.0
    assert bench.model_config("7b").head_bytes() == 2 * 32000 * 4096
