"""Trace-invariant checkers for EventTrace rows — a restatement of the
reference's own checkers (pkg/tests/helpers.py:80-151), used by the CPU tests
on reference-produced goldens and by the GPU tests on the engine's traces
(including the full 7B bench-config decode, tests/test_gpu_fulldepth.py).

Rows are (tick, stage, kind, position, token, verdict) with the kinds
ACTIVATION / DRAFT_TOKEN / FINAL_TOKEN / CHECK_TOKEN (pipesim.py:47-51).
"""

from collections import Counter

FORWARD_KINDS = ("ACTIVATION", "FINAL_TOKEN", "CHECK_TOKEN")
COMMIT_KINDS = ("FINAL_TOKEN", "CHECK_TOKEN")


def check_work_conservation(rows, n_stages: int, exit_stage: int) -> None:
    """helpers.py:80-92: one stage-forward per (tick, stage); commits only
    from the last stage; drafts only from the exit stage."""
    forwards = Counter()
    for r in rows:
        if r.kind in FORWARD_KINDS:
            forwards[(r.tick, r.stage)] += 1
        if r.kind in COMMIT_KINDS:
            assert r.stage == n_stages, f"commit from stage {r.stage}"
        if r.kind == "DRAFT_TOKEN":
            assert r.stage == exit_stage, f"draft from stage {r.stage}"
    for key, n in forwards.items():
        assert n == 1, f"stage ran {n} forwards at (tick, stage)={key}"


def check_commit_order(rows) -> None:
    """helpers.py:115-121: commits cover positions 1..K in order with
    non-decreasing ticks."""
    commits = [r for r in rows if r.kind in COMMIT_KINDS]
    for i, r in enumerate(commits, start=1):
        assert r.position == i, f"commit {i} carries position {r.position}"
    ticks = [r.tick for r in commits]
    assert ticks == sorted(ticks)


def check_flush_discipline(rows, relaunch_stage: int = 1) -> None:
    """helpers.py:124-151: commits land in position order, nothing works on a
    committed position, and after a rejection the first strictly later event
    is the relaunch of the next position at stage 1 (events sharing the
    rejection's tick are the other stages' parallel work and are exempt)."""
    committed = 0
    pending = None
    for r in rows:
        if r.kind in COMMIT_KINDS:
            assert r.position == committed + 1, f"commit carries position {r.position}, expected {committed + 1}"
            committed += 1
            if r.kind == "CHECK_TOKEN":
                pending = r.tick
        else:
            assert r.position > committed, f"{r.kind} at position {r.position} already committed"
            if pending is not None and r.tick > pending:
                assert r.position == committed + 1, f"stale in-flight position {r.position} survived a flush"
                assert r.stage == relaunch_stage
                pending = None


def check_all(rows, n_stages: int, exit_stage: int, comm_latency: int = 0) -> None:
    rows = list(rows)
    check_work_conservation(rows, n_stages, exit_stage)
    check_commit_order(rows)
    check_flush_discipline(rows)
