"""CPU Llama-style decoder oracle — TEST INFRASTRUCTURE ONLY.

The reference ships no neural network: its model is the hash ToyLM reached
through a 7-member duck-typed protocol (`n_layers`, `vocab`, `empty_digest`,
`extend_digest`, `advance_digest`, `dist_from_final_state`,
`exit_dist_from_states`; consumed at `pkg/src/specpipe/pipesim.py:306-315,
713-714, 735-743, 770, 401`). This module implements that protocol on a real
RMSNorm / RoPE / attention / SwiGLU decoder so the reference's own scheduler
(or `oracle/specpipe_port.py`) can drive it on the CPU and produce the
expected tokens, acceptance counts and traces for the GPU engine.

Digest = (trie node, layer). A trie node is one token at one position of one
(possibly speculative) prefix; it stores that position's K/V rows and the
hidden state at every layer boundary once forwarded. `advance_digest` only
relabels the layer, exactly like a pipeline stage handing its activation on;
the compute happens lazily when a head asks for a distribution.

Weights come from the counter-hash initialiser `init_tensor`, which the GPU
init kernel (`paper_2509_19368_b200/csrc/init.cu`) reproduces bit-for-bit:

    base  = mix64(mix64(seed ^ INIT_SALT) ^ tid)
    h_i   = mix64(base + (i+1)*GOLDEN)                  (i = logical row-major index)
    u_i   = (h_i >> 40) * 2^-24                          (exact fp32)
    w_i   = bf16_rne( fp32(2*u_i - 1) * fp32(sqrt(3/fan_in) * scale) )

so the weights are uniform with variance 1/fan_in (embedding: variance 1),
bf16-representable, and identical on CPU and GPU. Layers >= deep_from have
their residual writes (W_o, W_down) scaled by deep_scale: the misalignment
knob of SURVEY.md §0.4 (the transformer analogue of ToyLM's β,
`pkg/src/specpipe/toylm.py:10-13`). The exit head is a norm head: its own
RMSNorm followed by the tied LM head — or, with `exit_head_at=kE`, one more
decoder layer (init ids of layer index N, its own K/V per position) applied to
the layer-kE state before that norm head: the exit head of the paper's main
runs.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import asdict, dataclass

import numpy as np

from .specpipe_port import GOLDEN, M64, mix64, mix64_np

INIT_SALT = 0x5EED_B200_C0FF_EE01
TID_EMBED = 0xE0
TID_LM_HEAD = 0xE1
TID_WQ, TID_WK, TID_WV, TID_WO, TID_WGATE, TID_WUP, TID_WDOWN = 1, 2, 3, 4, 5, 6, 7


def layer_tid(layer: int, j: int) -> int:
    return ((layer + 1) << 8) | j


@dataclass(frozen=True)
class ModelShape:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab: int
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0

    def to_dict(self):
        return asdict(self)


def tiny_config(n_layers: int = 32) -> ModelShape:
    return ModelShape(n_layers, 64, 4, 4, 16, 176, 256)


def init_scale(fan_in: int, scale: float = 1.0) -> np.float32:
    return np.float32(math.sqrt(3.0 / fan_in) * scale)


def _bf16_round(x32: np.ndarray) -> np.ndarray:
    b = x32.view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return (b.astype(np.uint32) << 16).view(np.float32)


def _init_chunk(base: int, lo: int, hi: int, a32: np.float32) -> np.ndarray:
    idx = np.arange(lo + 1, hi + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = mix64_np(np.uint64(base) + idx * np.uint64(GOLDEN))
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    t = np.float32(2.0) * u - np.float32(1.0)
    return _bf16_round(t * a32)


_CINIT = []


def _cinit():
    """oracle/cinit.c (built by oracle/Makefile, `build()`): the same
    initialiser in C, ~50x faster for the 7B-70B shapes; None if not built."""
    if not _CINIT:
        import ctypes
        import os

        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle_cinit.so")
        lib = None
        if os.path.exists(path):
            try:
                lib = ctypes.CDLL(path)
                lib.oracle_init_tensor.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64,
                                                   ctypes.c_float, ctypes.c_int]
                lib.oracle_init_tensor.restype = ctypes.c_int
            except OSError:
                lib = None
        _CINIT.append(lib)
    return _CINIT[0]


def init_tensor(seed: int, tid: int, rows: int, cols: int, a32: np.float32,
                dtype=np.float64, threads: int = 8, use_c: bool = True) -> np.ndarray:
    """Logical [rows, cols] tensor from the counter hash (see module doc)."""
    base = mix64(mix64((seed ^ INIT_SALT) & M64) ^ tid)
    n = rows * cols
    lib = _cinit() if use_c else None
    if lib is not None:
        out32 = np.empty(n, dtype=np.float32)
        if lib.oracle_init_tensor(out32.ctypes.data, base, n, float(a32), max(1, threads)) != 0:
            raise RuntimeError("oracle_init_tensor failed")
        out = out32 if dtype == np.float32 else out32.astype(dtype)
        return out.reshape(rows, cols)
    out = np.empty(n, dtype=dtype)
    step = 1 << 22
    spans = [(lo, min(n, lo + step)) for lo in range(0, n, step)]

    def work(span):
        lo, hi = span
        out[lo:hi] = _init_chunk(base, lo, hi, a32)

    if len(spans) > 1 and threads > 1:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, spans))
    else:
        for s in spans:
            work(s)
    return out.reshape(rows, cols)


class Weights:
    def __init__(self, shape: ModelShape, seed: int, deep_scale: float = 1.0,
                 deep_from: int | None = None, dtype=np.float64, threads: int = 8, head_layer: bool = False):
        s = shape
        self.shape = s
        deep_from = s.n_layers if deep_from is None else deep_from
        qd, kvd = s.n_heads * s.head_dim, s.n_kv_heads * s.head_dim
        mk = lambda tid, r, c, a: init_tensor(seed, tid, r, c, a, dtype, threads)  # noqa: E731
        self.embed = mk(TID_EMBED, s.vocab, s.d_model, np.float32(math.sqrt(3.0)))
        self.lm_head = mk(TID_LM_HEAD, s.vocab, s.d_model, init_scale(s.d_model))
        self.layers = []
        for layer in range(s.n_layers):
            ds = deep_scale if layer >= deep_from else 1.0
            self.layers.append(dict(
                wq=mk(layer_tid(layer, TID_WQ), qd, s.d_model, init_scale(s.d_model)),
                wk=mk(layer_tid(layer, TID_WK), kvd, s.d_model, init_scale(s.d_model)),
                wv=mk(layer_tid(layer, TID_WV), kvd, s.d_model, init_scale(s.d_model)),
                wo=mk(layer_tid(layer, TID_WO), s.d_model, qd, init_scale(qd, ds)),
                wgate=mk(layer_tid(layer, TID_WGATE), s.ffn_dim, s.d_model, init_scale(s.d_model)),
                wup=mk(layer_tid(layer, TID_WUP), s.ffn_dim, s.d_model, init_scale(s.d_model)),
                wdown=mk(layer_tid(layer, TID_WDOWN), s.d_model, s.ffn_dim, init_scale(s.ffn_dim, ds)),
            ))
        self.head = None
        if head_layer:  # the exit head's decoder layer: layer index N, unscaled
            n = s.n_layers
            self.head = dict(
                wq=mk(layer_tid(n, TID_WQ), qd, s.d_model, init_scale(s.d_model)),
                wk=mk(layer_tid(n, TID_WK), kvd, s.d_model, init_scale(s.d_model)),
                wv=mk(layer_tid(n, TID_WV), kvd, s.d_model, init_scale(s.d_model)),
                wo=mk(layer_tid(n, TID_WO), s.d_model, qd, init_scale(qd)),
                wgate=mk(layer_tid(n, TID_WGATE), s.ffn_dim, s.d_model, init_scale(s.d_model)),
                wup=mk(layer_tid(n, TID_WUP), s.ffn_dim, s.d_model, init_scale(s.d_model)),
                wdown=mk(layer_tid(n, TID_WDOWN), s.d_model, s.ffn_dim, init_scale(s.ffn_dim)),
            )
        # norm weights are all ones (attn, mlp, final, exit)


def rope_tables(head_dim: int, theta: float, n_pos: int):
    """cos/sin [n_pos, head_dim/2] in float64 (the GPU reads these rounded to fp32)."""
    half = head_dim // 2
    inv = theta ** (-(2.0 * np.arange(half, dtype=np.float64)) / head_dim)
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


class _Node:
    __slots__ = ("parent", "tok", "pos", "kids", "k", "v", "hidden", "kh", "vh", "head_hidden")

    def __init__(self, parent, tok, pos):
        self.parent, self.tok, self.pos = parent, tok, pos
        self.kids = {}
        self.k = self.v = self.hidden = None
        self.kh = self.vh = self.head_hidden = None


class _PState:
    __slots__ = ("digest",)

    def __init__(self, d):
        self.digest = d


class TransformerOracle:
    """The reference's LM protocol on a CPU decoder (float64 by default)."""

    def __init__(self, shape: ModelShape, seed: int = 0, deep_scale: float = 1.0,
                 deep_from: int | None = None, dtype=np.float64, max_ctx: int = 4096,
                 threads: int = 8, weights: Weights | None = None, rope_fp32: bool = False,
                 exit_head_at: int | None = None, kv_bf16: bool = False):
        self.shape = shape
        # kv_bf16: K/V rows are stored rounded to bf16 (RNE), as the GPU's bf16
        # KV cache holds them; attention then reads the rounded rows
        self.kv_bf16 = kv_bf16
        self.n_layers, self.vocab = shape.n_layers, shape.vocab
        self.dtype = dtype
        self.exit_head_at = exit_head_at
        self.w = weights or Weights(shape, seed, deep_scale, deep_from, dtype, threads,
                                    head_layer=exit_head_at is not None)
        cos, sin = rope_tables(shape.head_dim, shape.rope_theta, max_ctx)
        if rope_fp32:
            cos, sin = cos.astype(np.float32), sin.astype(np.float32)
        self.cos, self.sin = cos.astype(dtype), sin.astype(dtype)
        self.root = _Node(None, None, -1)
        L, kvh, hd = shape.n_layers, shape.n_kv_heads, shape.head_dim
        self._K = np.zeros((L, max_ctx, kvh, hd), dtype)
        self._V = np.zeros((L, max_ctx, kvh, hd), dtype)
        self._owner = [None] * max_ctx  # node currently materialised at each position
        self._KH = np.zeros((max_ctx, kvh, hd), dtype)  # exit-head layer K/V
        self._VH = np.zeros((max_ctx, kvh, hd), dtype)
        self.margins = {"exit": math.inf, "final": math.inf}

    # ---- protocol --------------------------------------------------------
    def empty_digest(self):
        return (self.root, 0)

    def extend_digest(self, d, tok):
        node, layer = d
        if layer != 0:
            raise ValueError("extend_digest takes a layer-0 digest")
        if not 0 <= tok < self.vocab:
            raise ValueError(f"token {tok} outside vocab of {self.vocab}")
        kid = node.kids.get(tok)
        if kid is None:
            kid = node.kids[tok] = _Node(node, tok, node.pos + 1)
        return (kid, 0)

    def advance_digest(self, d, a, b):
        node, layer = d
        if layer != a or not 0 <= a <= b <= self.n_layers:
            raise ValueError(f"bad layer range {a}..{b} for digest at layer {layer}")
        return (node, b)

    def dist_from_final_state(self, state):
        node, layer = _dig(state)
        assert layer == self.n_layers
        z = self.final_logits(node)
        self._margin("final", z)
        return _Prob(_softmax(z))

    def exit_dist_from_states(self, final, exit_state):
        node, layer = _dig(exit_state)
        z = self.exit_logits(node, layer)
        self._margin("exit", z)
        return _Prob(_softmax(z))

    # ---- logits ----------------------------------------------------------
    def final_logits(self, node) -> np.ndarray:
        self._ensure(node)
        return self.w.lm_head @ self._rms(node.hidden[self.n_layers])

    def exit_logits(self, node, layer: int) -> np.ndarray:
        self._ensure(node)
        if self.exit_head_at is not None:
            assert layer == self.exit_head_at, (layer, self.exit_head_at)
            return self.w.lm_head @ self._rms(node.head_hidden)
        return self.w.lm_head @ self._rms(node.hidden[layer])

    def logits_for_prefix(self, tokens, layer=None):
        d = self.empty_digest()
        for t in tokens:
            d = self.extend_digest(d, t)
        node = d[0]
        return self.final_logits(node) if layer is None else self.exit_logits(node, layer)

    def path_logits(self, tokens, first: int, exit_layer: int):
        """Teacher-forced logits along ONE token path (one batched forward):
        for every prefix tokens[:j+1], j = first .. len-1, the exit-head
        logits (layer `exit_layer` state, or the exit head's layer) and the
        final-head logits, as float64 arrays [n, V] each. Row j predicts
        token j+1."""
        d = self.empty_digest()
        nodes = []
        for t in tokens:
            d = self.extend_digest(d, t)
            nodes.append(d[0])
        self._ensure(nodes[-1])
        sel = nodes[first:]
        if self.exit_head_at is not None:
            hx = np.stack([n.head_hidden for n in sel])
        else:
            hx = np.stack([n.hidden[exit_layer] for n in sel])
        hf = np.stack([n.hidden[self.n_layers] for n in sel])
        rms = lambda h: h / np.sqrt(np.mean(h * h, axis=1, keepdims=True) + self.shape.rms_eps)  # noqa: E731
        return ((rms(hx) @ self.w.lm_head.T).astype(np.float64),
                (rms(hf) @ self.w.lm_head.T).astype(np.float64))

    def margin_report(self):
        return {k: (None if math.isinf(v) else float(v)) for k, v in self.margins.items()}

    def _margin(self, key, z):
        top2 = np.partition(z, -2)[-2:]
        self.margins[key] = min(self.margins[key], float(top2[1] - top2[0]))

    # ---- forward ---------------------------------------------------------
    def _rms(self, x):
        s = self.shape
        return x / np.sqrt(np.mean(x * x) + s.rms_eps)

    def _ensure(self, node):
        if node.hidden is not None:
            return
        path = []
        n = node
        while n is not self.root and n.hidden is None:
            path.append(n)
            n = n.parent
        path.reverse()
        # materialise the already-forwarded ancestors' K/V rows (overwrite-by-position)
        anc = path[0].parent
        fix = []
        while anc is not self.root and self._owner[anc.pos] is not anc:
            fix.append(anc)
            anc = anc.parent
        for a in fix:
            self._K[:, a.pos] = a.k
            self._V[:, a.pos] = a.v
            if a.kh is not None:
                self._KH[a.pos] = a.kh
                self._VH[a.pos] = a.vh
            self._owner[a.pos] = a
        self._forward(path)

    def _layer(self, x, lw, Kst, Vst, p0, P, cos, sin):
        """One decoder layer on the path rows x [P, d] at positions p0..; K/V
        rows of the path go into Kst/Vst [pos, KV, hd] (the layer's cache)."""
        s = self.shape
        H, KV, hd = s.n_heads, s.n_kv_heads, s.head_dim
        rep = H // KV
        half = hd // 2
        scale = 1.0 / math.sqrt(hd)
        h = x / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + s.rms_eps)
        q = (h @ lw["wq"].T).reshape(P, H, hd)
        k = (h @ lw["wk"].T).reshape(P, KV, hd)
        v = (h @ lw["wv"].T).reshape(P, KV, hd)
        q = np.concatenate([q[..., :half] * cos - q[..., half:] * sin,
                            q[..., half:] * cos + q[..., :half] * sin], axis=-1)
        k = np.concatenate([k[..., :half] * cos - k[..., half:] * sin,
                            k[..., half:] * cos + k[..., :half] * sin], axis=-1)
        if self.kv_bf16:
            k = _bf16_round(k.astype(np.float32)).astype(self.dtype)
            v = _bf16_round(np.ascontiguousarray(v, dtype=np.float32)).astype(self.dtype)
        Kst[p0:p0 + P] = k
        Vst[p0:p0 + P] = v
        Kc = Kst[:p0 + P]  # [T, KV, hd]
        Vc = Vst[:p0 + P]
        causal = np.tril(np.ones((P, P), bool))
        o = np.empty((P, H, hd), self.dtype)
        for hh in range(H):
            kh = hh // rep
            sc = (q[:, hh, :] @ Kc[:, kh, :].T) * scale  # [P, T]
            if P > 1:
                mask = np.ones((P, p0 + P), bool)
                mask[:, p0:] = causal
                sc = np.where(mask, sc, -np.inf)
            sc = sc - sc.max(axis=1, keepdims=True)
            e = np.exp(sc)
            o[:, hh, :] = (e @ Vc[:, kh, :]) / e.sum(axis=1, keepdims=True)
        x = x + o.reshape(P, H * hd) @ lw["wo"].T
        h = x / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + s.rms_eps)
        g = h @ lw["wgate"].T
        u = h @ lw["wup"].T
        a = g / (1.0 + np.exp(-g)) * u
        return x + a @ lw["wdown"].T, k, v

    def _forward(self, path):
        s, w = self.shape, self.w
        KV, hd = s.n_kv_heads, s.head_dim
        p0 = path[0].pos
        P = len(path)
        pos = np.arange(p0, p0 + P)
        x = w.embed[[n.tok for n in path]].astype(self.dtype)  # [P, d]
        hid = [x.copy()]
        ks = np.empty((s.n_layers, P, KV, hd), self.dtype)
        vs = np.empty_like(ks)
        cos, sin = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        for li, lw in enumerate(w.layers):
            x, ks[li], vs[li] = self._layer(x, lw, self._K[li], self._V[li], p0, P, cos, sin)
            hid.append(x.copy())
        head = None
        if self.exit_head_at is not None:  # the exit head's layer on the layer-kE states
            head, kh, vh = self._layer(hid[self.exit_head_at].copy(), w.head, self._KH, self._VH, p0, P, cos, sin)
        for i, n in enumerate(path):
            n.k, n.v = ks[:, i].copy(), vs[:, i].copy()
            n.hidden = [hl[i] for hl in hid]
            if head is not None:
                n.kh, n.vh, n.head_hidden = kh[i].copy(), vh[i].copy(), head[i]
            self._owner[n.pos] = n


class _Prob:
    """Duck-typed stand-in for the reference ProbVec (.probs, len, getitem)."""

    __slots__ = ("probs",)

    def __init__(self, p):
        self.probs = p

    def __len__(self):
        return len(self.probs)

    def __getitem__(self, i):
        return float(self.probs[i])


def _softmax(z):
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max())
    return e / e.sum()


def _dig(s):
    return s.digest if hasattr(s, "digest") else s
