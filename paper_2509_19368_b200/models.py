"""Device-resident models the decode engine runs.

* ToyLM — same constructor and validation as the reference model
  (pkg/src/specpipe/toylm.py:55-68); its digest chain, hashed logits and
  exit-head noise run on the GPU (csrc/toylm.cu), bit-exact with the
  reference.
* TransformerLM — a Llama-style decoder (RMSNorm, RoPE, paged-KV attention,
  SwiGLU, tied early-exit norm head) with bf16 weights initialised on the GPU
  by the counter-hash initialiser that oracle/transformer.py reproduces on
  the CPU. It implements no Python-side compute: every forward is a kernel.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib

LAYOUT_TC_TILED = 16  # include/ppsd.h PPSD_LAYOUT_TC_TILED
INIT_SALT = 0x5EED_B200_C0FF_EE01  # keep in sync with csrc/engine.cu ppsd_init_weight
TID_EMBED, TID_LM_HEAD = 0xE0, 0xE1
TID_WQ, TID_WK, TID_WV, TID_WO, TID_WGATE, TID_WUP, TID_WDOWN = 1, 2, 3, 4, 5, 6, 7


def layer_tid(layer: int, j: int) -> int:
    return ((layer + 1) << 8) | j


def init_scale(fan_in: int, scale: float = 1.0) -> float:
    """sqrt(3/fan_in)*scale rounded to fp32: uniform init with variance 1/fan_in."""
    return float(np.float32(math.sqrt(3.0 / fan_in) * scale))


@dataclass(frozen=True)
class ToyLM:
    n_layers: int
    vocab: int
    seed: int
    misalignment: float = 0.0

    def __post_init__(self):
        if self.n_layers < 1:
            raise ValueError("n_layers must be >= 1")
        if self.vocab < 2:
            raise ValueError("vocab must be >= 2")
        if self.misalignment < 0.0:
            raise ValueError("misalignment must be non-negative")

    def model_desc(self, max_ctx: int) -> _lib.ModelDesc:
        return _lib.ModelDesc(kind=_lib.MODEL_TOYLM, n_layers=self.n_layers, vocab=self.vocab,
                              max_ctx=max_ctx, toy_seed=self.seed & ((1 << 64) - 1),
                              toy_misalignment=float(self.misalignment))

    # ---- measured alignment (toylm.py:153-192), evaluated on the GPU ----

    EVAL_PREFIX_LEN = 8  # toylm.py:32

    def _alignment(self, exit_depth: int, n_prefixes: int, eval_seed: int | None):
        from .decode import toy_alignment
        from .rng import RngStream, derive_seed

        if n_prefixes < 1:
            raise ValueError("n_prefixes must be >= 1")
        if eval_seed is None:
            eval_seed = derive_seed(self.seed, "empirical-alpha")
        stream = RngStream(eval_seed)
        prefixes = [[stream.randbelow(self.vocab) for _ in range(self.EVAL_PREFIX_LEN)]
                    for _ in range(n_prefixes)]
        return toy_alignment(self, exit_depth, prefixes)

    def empirical_alpha(self, exit_depth: int, n_prefixes: int, eval_seed: int | None = None) -> float:
        """Mean sum(min(p, q)) over seeded random prefixes: the acceptance
        rate of sampling-mode verification (toylm.py:165-179)."""
        minsum, _ = self._alignment(exit_depth, n_prefixes, eval_seed)
        acc = 0.0
        for v in minsum:  # the reference's left-to-right accumulation
            acc += float(v)
        return acc / n_prefixes

    def greedy_agreement(self, exit_depth: int, n_prefixes: int, eval_seed: int | None = None) -> float:
        """Fraction of seeded random prefixes whose exit-head and full-model
        argmax agree: the greedy-mode acceptance rate (toylm.py:181-192)."""
        _, agree = self._alignment(exit_depth, n_prefixes, eval_seed)
        return int(sum(int(a) for a in agree)) / n_prefixes


@dataclass(frozen=True)
class TransformerConfig:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0
    kv_dtype: str = "bf16"
    max_ctx: int = 1024
    name: str = field(default="custom", compare=False)

    def __post_init__(self):
        if self.kv_dtype not in ("bf16", "fp32"):
            raise ValueError("kv_dtype must be 'bf16' or 'fp32'")
        if self.n_heads % self.n_kv_heads:
            raise ValueError("n_heads must be a multiple of n_kv_heads")

    @staticmethod
    def tiny(n_layers: int = 32) -> "TransformerConfig":
        """The small parity config (d=64, 4 heads, ffn 176, V=256, fp32 KV)."""
        return TransformerConfig(n_layers, 64, 4, 4, 16, 176, 256, kv_dtype="fp32", name="tiny")

    @staticmethod
    def llama2_7b(**kw) -> "TransformerConfig":
        return replace(TransformerConfig(32, 4096, 32, 32, 128, 11008, 32000, name="llama2-7b"), **kw)

    @staticmethod
    def llama2_13b(**kw) -> "TransformerConfig":
        return replace(TransformerConfig(40, 5120, 40, 40, 128, 13824, 32000, name="llama2-13b"), **kw)

    @staticmethod
    def llama2_70b(**kw) -> "TransformerConfig":
        return replace(TransformerConfig(80, 8192, 64, 8, 128, 28672, 32000, name="llama2-70b"), **kw)

    def layer_bytes(self) -> int:
        d, qd, kvd = self.d_model, self.n_heads * self.head_dim, self.n_kv_heads * self.head_dim
        return 2 * ((qd + 2 * kvd) * d + d * qd + 2 * self.ffn_dim * d + d * self.ffn_dim)

    def head_bytes(self) -> int:
        return 2 * self.vocab * self.d_model

    def kv_bytes_per_token_layer(self) -> int:
        return 2 * self.n_kv_heads * self.head_dim * (2 if self.kv_dtype == "bf16" else 4)

    def to_desc(self) -> _lib.ModelDesc:
        return _lib.ModelDesc(kind=_lib.MODEL_TRANSFORMER, n_layers=self.n_layers, vocab=self.vocab,
                              d_model=self.d_model, n_heads=self.n_heads, n_kv_heads=self.n_kv_heads,
                              head_dim=self.head_dim, ffn_dim=self.ffn_dim, rms_eps=self.rms_eps,
                              rope_theta=self.rope_theta, kv_bf16=int(self.kv_dtype == "bf16"),
                              max_ctx=self.max_ctx)


def rope_tables(head_dim: int, theta: float, n_pos: int):
    """cos/sin [n_pos, head_dim/2], computed in float64 then rounded to fp32."""
    half = head_dim // 2
    inv = theta ** (-(2.0 * np.arange(half, dtype=np.float64)) / head_dim)
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def tc_layout(rows: int, cols: int) -> tuple[int, int]:
    """(JS, KP) of the TC-tiled layout of a [rows][cols] matrix (csrc/kernels.cuh tc_layout)."""
    kp = (cols + 63) // 64 * 64
    nsl = kp // 64
    js = 4 if nsl % 4 == 0 else 2 if nsl % 2 == 0 else 1
    return js, kp


def tc_tile(w: np.ndarray) -> np.ndarray:
    """A row-major [rows][cols] matrix in the TC-tiled layout the tensor-core
    GEMV streams: flat, cols padded with zeros to a multiple of
    64, element (r, k) at csrc/kernels.cuh tc_offset. For loading checkpoints;
    the random-init weights are written tiled on the GPU (ppsd_init_weight)."""
    rows, cols = w.shape
    if rows % 8 or cols % 8:
        raise ValueError("TC-tiled matrices need rows and cols multiples of 8")
    js, kp = tc_layout(rows, cols)
    g = rows // 8
    out = np.zeros(rows * kp, dtype=w.dtype)
    r = np.arange(rows)[:, None]
    k = np.arange(cols)[None, :]
    slab, rr, c, e = k // 64, r % 8, (k % 64) // 8, k % 8
    off = (((((slab // js) * g + r // 8) * js + slab % js) * 8 + rr) * 64) + ((c ^ rr) * 8) + e
    out[off.ravel()] = w.ravel()
    return out


class TransformerLM:
    """Random-init Llama-shaped decoder resident on one GPU.

    deep_scale scales the residual writes (W_o, W_down) of layers >=
    deep_from: the deterministic misalignment knob that sets how often the
    early-exit head agrees with the final head. `layers`
    restricts materialisation to a [lo, hi) layer range (one pipeline rank).
    `schedule` picks how a single-device engine executes the machine
    ('auto' | 'pipelined' | 'folded', include/ppsd.h PPSD_SCHEDULE_*); every
    schedule returns the same tokens, metrics and trace.
    """

    schedule = "auto"

    def __init__(self, config: TransformerConfig, seed: int = 0, deep_scale: float = 1.0,
                 deep_from: int | None = None, device=None, layers: tuple[int, int] | None = None,
                 need_embed: bool = True, need_head: bool = True, exit_head: str = "norm"):
        import torch

        if exit_head not in ("norm", "layer"):
            raise ValueError(f"exit_head must be 'norm' or 'layer', got {exit_head!r}")
        self.config = config
        self.exit_head = exit_head
        self.n_layers, self.vocab = config.n_layers, config.vocab
        self.seed, self.deep_scale = seed, float(deep_scale)
        self.deep_from = config.n_layers if deep_from is None else deep_from
        self.device = _lib.require_cuda(device if device is None or isinstance(device, int)
                                        else torch.device(device).index)
        L = _lib.lib()
        c = config
        lo, hi = layers if layers is not None else (0, c.n_layers)
        self.layer_range = (lo, hi)
        qd, kvd = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
        dev = self.device
        bf = torch.bfloat16
        self._keep = []
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream

            pools = {}

            def init(rows, cols, layout, tids, scales, tiled=True, pool=None):
                # GEMV matrices live in the tensor-core GEMV's TC-tiled layout
                # (include/ppsd.h PPSD_LAYOUT_TC_TILED); the embedding is gathered by
                # rows and stays plain. pool: the layers' matrices of one kind are
                # slices of one allocation, so they sit at a fixed stride (the GEMV
                # computes their address instead of loading it)
                n = C.c_int64(0)
                _lib.check(L.ppsd_weight_elems(int(tiled), rows, cols, C.byref(n)), "weight_elems")
                if pool is not None:
                    buf, step, used = pools.get(pool, (None, 0, 0))
                    if buf is None:
                        step = (n.value + 127) // 128 * 128  # 256-byte aligned slices
                        buf = torch.empty(step * (hi - lo), dtype=bf, device=dev)
                    t = buf[used * step:used * step + n.value]
                    pools[pool] = (buf, step, used + 1)
                else:
                    t = torch.empty(n.value, dtype=bf, device=dev)
                tid_arr = (C.c_uint64 * 3)(*(list(tids) + [0] * (3 - len(tids))))
                sc_arr = (C.c_float * 3)(*(list(scales) + [0.0] * (3 - len(scales))))
                lay = layout | (LAYOUT_TC_TILED if tiled else 0)
                _lib.check(L.ppsd_init_weight(C.c_void_p(t.data_ptr()), lay, rows, cols,
                                              seed & ((1 << 64) - 1), tid_arr, sc_arr, c.n_heads,
                                              c.n_kv_heads, c.head_dim, C.c_void_p(stream)),
                           "init")
                return t

            s_d = init_scale(c.d_model)
            self.embed = init(c.vocab, c.d_model, 0, [TID_EMBED], [float(np.float32(math.sqrt(3.0)))],
                              tiled=False) \
                if need_embed else None
            self.lm_head = init(c.vocab, c.d_model, 0, [TID_LM_HEAD], [s_d]) if need_head else None
            ones = lambda: torch.ones(c.d_model, dtype=torch.float32, device=dev)  # noqa: E731
            self.final_norm, self.exit_norm = ones(), ones()
            self.w_qkv, self.w_o, self.w_gu, self.w_down = [None] * c.n_layers, [None] * c.n_layers, \
                [None] * c.n_layers, [None] * c.n_layers
            self.attn_norm, self.mlp_norm = [None] * c.n_layers, [None] * c.n_layers
            for layer in range(lo, hi):
                ds = self.deep_scale if layer >= self.deep_from else 1.0
                self.w_qkv[layer] = init(qd + 2 * kvd, c.d_model, 1,
                                         [layer_tid(layer, TID_WQ), layer_tid(layer, TID_WK),
                                          layer_tid(layer, TID_WV)], [s_d, s_d, s_d], pool="qkv")
                self.w_o[layer] = init(c.d_model, qd, 0, [layer_tid(layer, TID_WO)], [init_scale(qd, ds)],
                                       pool="o")
                self.w_gu[layer] = init(2 * c.ffn_dim, c.d_model, 2,
                                        [layer_tid(layer, TID_WGATE), layer_tid(layer, TID_WUP)], [s_d, s_d],
                                        pool="gu")
                self.w_down[layer] = init(c.d_model, c.ffn_dim, 0, [layer_tid(layer, TID_WDOWN)],
                                          [init_scale(c.ffn_dim, ds)], pool="down")
                self.attn_norm[layer], self.mlp_norm[layer] = ones(), ones()
            self.exit_layer_w = None
            if exit_head == "layer":  # the exit head's decoder layer: layer index N in the init ids
                n = c.n_layers
                self.exit_layer_w = dict(
                    qkv=init(qd + 2 * kvd, c.d_model, 1,
                             [layer_tid(n, TID_WQ), layer_tid(n, TID_WK), layer_tid(n, TID_WV)], [s_d, s_d, s_d]),
                    o=init(c.d_model, qd, 0, [layer_tid(n, TID_WO)], [init_scale(qd)]),
                    gu=init(2 * c.ffn_dim, c.d_model, 2, [layer_tid(n, TID_WGATE), layer_tid(n, TID_WUP)],
                            [s_d, s_d]),
                    down=init(c.d_model, c.ffn_dim, 0, [layer_tid(n, TID_WDOWN)], [init_scale(c.ffn_dim)]),
                    attn_norm=ones(), mlp_norm=ones())
            cos, sin = rope_tables(c.head_dim, c.rope_theta, c.max_ctx)
            self.rope_cos = torch.from_numpy(cos).to(dev)
            self.rope_sin = torch.from_numpy(sin).to(dev)
            torch.cuda.synchronize(dev)

    def model_desc(self, max_ctx: int | None = None) -> _lib.ModelDesc:
        d = self.config.to_desc()
        d.exit_head_layer = int(self.exit_head == "layer")
        return d

    def weights_struct(self) -> _lib.Weights:
        n = self.config.n_layers
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731

        def arr(ts):
            a = (C.c_void_p * n)(*[ptr(t) for t in ts])
            self._keep.append(a)
            return a

        xl = _lib.LayerWeights()
        if self.exit_layer_w is not None:
            X = self.exit_layer_w
            xl = _lib.LayerWeights(qkv=ptr(X["qkv"]), o=ptr(X["o"]), gu=ptr(X["gu"]), down=ptr(X["down"]),
                                   attn_norm=ptr(X["attn_norm"]), mlp_norm=ptr(X["mlp_norm"]))
        return _lib.Weights(embed=ptr(self.embed), lm_head=ptr(self.lm_head),
                            final_norm=ptr(self.final_norm), exit_norm=ptr(self.exit_norm),
                            w_qkv=arr(self.w_qkv), w_o=arr(self.w_o), w_gu=arr(self.w_gu),
                            w_down=arr(self.w_down), attn_norm=arr(self.attn_norm),
                            mlp_norm=arr(self.mlp_norm), rope_cos=ptr(self.rope_cos),
                            rope_sin=ptr(self.rope_sin), exit_layer=xl)

    def weight_bytes(self) -> int:
        lo, hi = self.layer_range
        return (hi - lo) * self.config.layer_bytes() + self.config.head_bytes()
