"""The tensor-core GEMV (csrc/tcgemv.cu) as a plain matrix-vector product.

y_v = W x_v for the O and down projections through the shipped kernel
(ppsd_debug_matvec: residual epilogue into a zeroed hidden state), checked
against float64 numpy on the oracle's own weights (oracle/transformer.py
init_tensor, the counter hash the device initialiser reproduces), and for
batch invariance: a vector's row sums are bit-identical whatever the number
of vectors in the weight pass and whichever plan (decode tick / batched) runs
it — the property PPSD == AR rests on.

Tolerance: the activations enter the MMA as an exact three-way bf16 split and
the weights are bf16, so every product is exact; only the fp32 accumulation
order differs from float64: |dy| <= 1e-5 * sum_k |W x| + 1e-6.
"""
import numpy as np
import pytest

ppsd = pytest.importorskip("paper_2509_19368_b200")

pytestmark = pytest.mark.gpu

SHAPES = {
    "tiny": dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=4, head_dim=16, ffn_dim=176, vocab=256),
    "l7b": dict(n_layers=2, d_model=4096, n_heads=32, n_kv_heads=32, head_dim=128, ffn_dim=11008,
                vocab=32000),
    "mid_gqa": dict(n_layers=2, d_model=1024, n_heads=16, n_kv_heads=4, head_dim=64, ffn_dim=2816,
                    vocab=4096),
}


@pytest.fixture(scope="module", params=list(SHAPES))
def engine(request):
    from oracle.transformer import init_scale, init_tensor, layer_tid
    from paper_2509_19368_b200.models import TID_WDOWN, TID_WO

    sh = SHAPES[request.param]
    config = ppsd.TransformerConfig(**sh, kv_dtype="bf16", max_ctx=128)
    lm = ppsd.TransformerLM(config, seed=7)
    eng = ppsd.engine_for(lm, ppsd.PipelineConfig(config.n_layers, 1))
    layer = config.n_layers - 1
    qd = config.n_heads * config.head_dim
    W = {1: init_tensor(7, layer_tid(layer, TID_WO), config.d_model, qd, init_scale(qd)),
         3: init_tensor(7, layer_tid(layer, TID_WDOWN), config.d_model, config.ffn_dim,
                        init_scale(config.ffn_dim))}
    return eng, layer, W


@pytest.mark.parametrize("which", [1, 3])
def test_matvec_vs_float64(engine, which):
    eng, layer, W = engine
    Wm = W[which]
    rng = np.random.default_rng(which)
    for nv, batched in ((1, False), (5, False), (16, True)):
        x = rng.standard_normal((nv, Wm.shape[1])).astype(np.float32)
        y = eng.debug_matvec(which, layer, x, batched)
        want = x.astype(np.float64) @ Wm.T
        bound = 1e-5 * (np.abs(x.astype(np.float64)) @ np.abs(Wm).T) + 1e-6
        bad = np.abs(y - want) > bound
        assert not bad.any(), f"nv={nv}: {bad.sum()} rows off, max |dy| {np.abs(y - want).max():.3e}"


@pytest.mark.parametrize("which", [1, 3])
def test_matvec_batch_invariant(engine, which):
    eng, layer, W = engine
    rng = np.random.default_rng(10 + which)
    x = rng.standard_normal((16, W[which].shape[1])).astype(np.float32)
    solo = np.stack([eng.debug_matvec(which, layer, x[v:v + 1], False)[0] for v in range(16)])
    for nv, batched in ((2, False), (5, False), (1, True), (4, True), (11, True), (16, True)):
        got = eng.debug_matvec(which, layer, x[:nv], batched)
        assert np.array_equal(got.view(np.uint32), solo[:nv].view(np.uint32)), (nv, batched)
    # a vector's result does not depend on its column in the pass
    rot = np.roll(x[:5], 2, axis=0)
    got = eng.debug_matvec(which, layer, rot, False)
    assert np.array_equal(got.view(np.uint32), np.roll(solo[:5], 2, axis=0).view(np.uint32))
