"""CLI subcommands that need no GPU (`analytic`, `--dump-config`, config
errors) against the reference transcripts (tests/golden/cli_harness.json)."""

import pytest

from test_cli_gpu import HARNESS, _host_only, _run_cli


@pytest.mark.parametrize("case", [c for c in HARNESS["commands"] if _host_only(c["argv"], c["returncode"])],
                         ids=lambda c: " ".join(c["argv"][:3]))
def test_cli_host_commands_match_reference(case, tmp_path):
    _run_cli(case, tmp_path)
