"""B200-native greedy PPSD (pipeline-parallel self-speculative) decoding.

Drop-in for the decode path of the reference `specpipe` package
(pkg/src/specpipe/__init__.py:59-106 names): the same PipelineConfig,
decode_ppsd / decode_autoregressive / simulate_ppsd signatures, RunMetrics
and EventTrace, executed by hand-written sm_100a kernels in libppsd.so.
"""

__version__ = "0.1.0"

from .analytic import (SpeedupParams, eesd_speedup, expected_accept_len, n_stages,
                       ppsd_over_eesd_lambda, ppsd_reference_speedup, ppsd_speedup)
from .decode import (Engine, decode_autoregressive, decode_eesd, decode_ppsd, engine_for,
                     simulate_autoregressive, simulate_eesd, simulate_ppsd)
from .models import ToyLM, TransformerConfig, TransformerLM, tc_tile
from .pipeline import (ACTIVATION, CHECK_TOKEN, DRAFT_TOKEN, FINAL_TOKEN, TRACE_HEADER,
                       AcceptanceOracle, EventTrace, OracleMode, PipelineConfig, RunMetrics,
                       StageMessage, TraceRow, default_prompt, partition_stages, steady_state_view)
from .rng import RngStream, derive_seed, mix64

__all__ = [
    "ACTIVATION", "CHECK_TOKEN", "DRAFT_TOKEN", "FINAL_TOKEN", "TRACE_HEADER",
    "AcceptanceOracle", "Engine", "EventTrace", "OracleMode", "PipelineConfig", "RngStream",
    "RunMetrics", "SpeedupParams", "StageMessage", "ToyLM", "TraceRow", "TransformerConfig",
    "TransformerLM", "tc_tile", "decode_autoregressive", "decode_eesd", "decode_ppsd", "default_prompt", "derive_seed",
    "eesd_speedup", "engine_for", "expected_accept_len", "mix64", "n_stages", "partition_stages",
    "ppsd_over_eesd_lambda", "ppsd_reference_speedup", "ppsd_speedup", "simulate_autoregressive",
    "simulate_eesd", "simulate_ppsd", "steady_state_view",
]
