"""ctypes binding of libppsd.so (include/ppsd.h).

The shipped decode path has exactly one implementation: the sm_100a kernels
in this library. There is no CPU fallback — if the library or a CUDA device
is missing, `lib()` raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# PPSD_LIB: another build of the library (A/B experiments, e.g. tools/quick_decode.py)
LIB_PATH = os.environ.get("PPSD_LIB") or os.path.join(HERE, "libppsd.so")

PPSD_OK, PPSD_EINVAL, PPSD_ECUDA, PPSD_ESTATE, PPSD_EUNSUPPORTED = 0, -1, -2, -3, -4
MODEL_BERNOULLI, MODEL_TOYLM, MODEL_TRANSFORMER = 0, 1, 2
# execution schedules of a single-device engine (include/ppsd.h PPSD_SCHEDULE_*)
SCHEDULES = {"auto": 0, "pipelined": 1, "folded": 2}


def schedule_name(code: int) -> str:
    """The schedule a decode ran (ppsd_metrics.schedule)."""
    return {v: k for k, v in SCHEDULES.items()}.get(code, "pipelined")


class ModelDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("n_layers", C.c_int32), ("vocab", C.c_int32),
        ("d_model", C.c_int32), ("n_heads", C.c_int32), ("n_kv_heads", C.c_int32),
        ("head_dim", C.c_int32), ("ffn_dim", C.c_int32),
        ("rms_eps", C.c_float), ("rope_theta", C.c_float),
        ("kv_bf16", C.c_int32), ("max_ctx", C.c_int32),
        ("toy_seed", C.c_uint64), ("toy_misalignment", C.c_double), ("exit_head_layer", C.c_int32),
    ]


class LayerWeights(C.Structure):
    _fields_ = [("qkv", C.c_void_p), ("o", C.c_void_p), ("gu", C.c_void_p), ("down", C.c_void_p),
                ("attn_norm", C.c_void_p), ("mlp_norm", C.c_void_p)]


class Weights(C.Structure):
    _fields_ = [
        ("embed", C.c_void_p), ("lm_head", C.c_void_p),
        ("final_norm", C.c_void_p), ("exit_norm", C.c_void_p),
        ("w_qkv", C.POINTER(C.c_void_p)), ("w_o", C.POINTER(C.c_void_p)),
        ("w_gu", C.POINTER(C.c_void_p)), ("w_down", C.POINTER(C.c_void_p)),
        ("attn_norm", C.POINTER(C.c_void_p)), ("mlp_norm", C.POINTER(C.c_void_p)),
        ("rope_cos", C.c_void_p), ("rope_sin", C.c_void_p), ("exit_layer", LayerWeights),
    ]


class PipelineDesc(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("exit_depth", C.c_int32), ("exit_stage", C.c_int32),
        ("comm_latency", C.c_int32), ("stage_lo", C.c_int32), ("stage_hi", C.c_int32),
        ("device", C.c_int32), ("schedule", C.c_int32),
    ]


class Metrics(C.Structure):
    _fields_ = [
        ("committed_tokens", C.c_int64), ("ticks", C.c_int64), ("accepts", C.c_int64),
        ("rejects", C.c_int64), ("alpha_valid", C.c_int32),
        ("alpha_all_measured", C.c_double), ("throughput", C.c_double),
        ("speedup_vs_ar", C.c_double), ("decode_ms", C.c_double), ("prefill_ms", C.c_double),
        ("gpu_launches", C.c_int64), ("schedule", C.c_int32), ("deep_batches", C.c_int64),
        ("deep_vectors", C.c_int64), ("deep_pos_sum", C.c_int64), ("comb_heads", C.c_int64),
    ]


class TraceRowC(C.Structure):
    _fields_ = [("tick", C.c_int32), ("stage", C.c_int32), ("kind", C.c_int32),
                ("position", C.c_int32), ("token", C.c_int32), ("verdict", C.c_int32)]


EXPORTS = {
    "ppsd_last_error": (C.c_char_p, []),
    "ppsd_build_info": (C.c_char_p, []),
    "ppsd_engine_create": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(Weights),
                                     C.POINTER(PipelineDesc), C.c_void_p, C.POINTER(C.c_void_p)]),
    "ppsd_engine_destroy": (C.c_int, [C.c_void_p]),
    "ppsd_decode": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.POINTER(C.c_int32), C.c_int32,
                              C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(Metrics),
                              C.POINTER(TraceRowC), C.c_int64, C.POINTER(C.c_int64)]),
    "ppsd_set_schedule": (C.c_int, [C.c_void_p, C.c_int32]),
    "ppsd_toy_alignment": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    "ppsd_get_schedule": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]),
    "ppsd_decode_ar": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.POINTER(C.c_int32), C.c_int32,
                                 C.c_int32, C.POINTER(C.c_int32), C.POINTER(Metrics)]),
    "ppsd_decode_eesd": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                   C.POINTER(C.c_int32), C.c_int32, C.POINTER(Metrics),
                                   C.POINTER(TraceRowC), C.c_int64, C.POINTER(C.c_int64)]),
    "ppsd_decode_eesd_mode": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(C.c_int32),
                                        C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.POINTER(Metrics),
                                        C.POINTER(TraceRowC), C.c_int64, C.POINTER(C.c_int64)]),
    "ppsd_simulate_eesd": (C.c_int, [C.c_void_p, C.c_int32, C.c_double, C.c_uint64, C.c_int32,
                                     C.POINTER(Metrics), C.POINTER(TraceRowC), C.c_int64,
                                     C.POINTER(C.c_int64)]),
    "ppsd_simulate": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64, C.c_int32, C.c_int32,
                                C.POINTER(Metrics), C.POINTER(TraceRowC), C.c_int64,
                                C.POINTER(C.c_int64)]),
    "ppsd_exchange_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_void_p)]),
    "ppsd_step_mode": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64]),
    "ppsd_step_begin": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "ppsd_prefill_steps": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "ppsd_prefill_compute": (C.c_int, [C.c_void_p]),
    "ppsd_step_compute": (C.c_int, [C.c_void_p]),
    "ppsd_step_finish": (C.c_int, [C.c_void_p]),
    "ppsd_step_poll": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64)]),
    "ppsd_step_end": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(Metrics),
                                C.POINTER(TraceRowC), C.c_int64, C.POINTER(C.c_int64)]),
    "ppsd_p2p_prepare": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ppsd_p2p_connect": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p),
                                   C.POINTER(C.c_int32)]),
    "ppsd_p2p_decode": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(C.c_int32), C.POINTER(Metrics), C.POINTER(TraceRowC), C.c_int64,
                                  C.POINTER(C.c_int64)]),
    "ppsd_debug_matvec": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                    C.POINTER(C.c_float), C.POINTER(C.c_float)]),
    "ppsd_debug_tc_trace": (C.c_int, [C.c_int32, C.POINTER(C.c_uint64)]),
    "ppsd_tc_offset": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_int64)]),
    "ppsd_weight_elems": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, C.POINTER(C.c_int64)]),
    "ppsd_init_weight": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_uint64,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_float), C.c_int32, C.c_int32,
                                   C.c_int32, C.c_void_p]),
    "ppsd_read_logits": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_float)]),
    "ppsd_set_logits_tap": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "ppsd_probe_attn": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]),
    "ppsd_probe_gemv": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

_lock = threading.Lock()
_lib = None


class PpsdError(RuntimeError):
    pass


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libppsd.so and bind every export of include/ppsd.h (no GPU needed)."""
    if not os.path.exists(path):
        raise PpsdError(
            f"{path} is missing: build it with `make -C paper_2509_19368_b200/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            _lib = load_library()
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == PPSD_OK:
        return
    msg = (lib().ppsd_last_error() or b"").decode(errors="replace")
    if rc == PPSD_EINVAL:
        raise ValueError(msg)
    if rc == PPSD_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise PpsdError(f"{what}: {msg} (status {rc})")


def require_cuda(device=None):
    import torch

    if not torch.cuda.is_available():
        raise PpsdError("the B200 PPSD engine needs a CUDA device (sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device() if device is None else device)
