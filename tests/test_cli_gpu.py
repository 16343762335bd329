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
