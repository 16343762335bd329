"""`python -m paper_2509_19368_b200 decode` output equals `specpipe decode`'s
(reference transcripts recorded in tests/golden/cli_decode.json)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "cli_decode.json")) as fh:
    CASES = json.load(fh)["cases"]


@pytest.mark.parametrize("case", CASES, ids=lambda c: " ".join(c["argv"][-4:]))
def test_cli_decode_matches_reference(case):
    out = subprocess.run([sys.executable, "-m", "paper_2509_19368_b200", *case["argv"]], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == case["returncode"], out.stderr
    assert out.stdout == case["stdout"]


with open(os.path.join(GOLDEN, "cli_harness.json")) as fh:
    HARNESS = json.load(fh)["cases"][0]


def _host_only(argv, rc):
    return rc != 0 or argv[0] == "analytic" or "--dump-config" in argv


def _run_cli(case, tmp_path):
    paths = {"config_json": str(tmp_path / "config.json"), "sweep_json": str(tmp_path / "sweep.json")}
    with open(paths["config_json"], "w") as fh:
        fh.write(HARNESS["config_json"])  # file texts (axis order matters)
    with open(paths["sweep_json"], "w") as fh:
        fh.write(HARNESS["sweep_json"])
    argv = [a.format(**paths) for a in case["argv"]]
    out = subprocess.run([sys.executable, "-m", "paper_2509_19368_b200", *argv], cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == case["returncode"], out.stderr
    assert out.stdout == case["stdout"]
    assert out.stderr == case["stderr"]


@pytest.mark.parametrize("case", [c for c in HARNESS["commands"] if not _host_only(c["argv"], c["returncode"])],
                         ids=lambda c: " ".join(c["argv"][:3]))
def test_cli_harness_matches_reference(case, tmp_path):
    """`run` / `sweep` on the GPU tick machine print what `specpipe run|sweep` print."""
    _run_cli(case, tmp_path)
