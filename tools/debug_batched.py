import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

def child(chunk):
    os.environ["PPSD_PREFILL_CHUNK"] = str(chunk)
    import paper_2509_19368_b200 as ppsd
    name = sys.argv[2]
    shapes = {"mid": (8, 1024, 16, 4, 64, 2816, 4096), "l7b": (2, 4096, 32, 32, 128, 11008, 32000)}
    n, d, H, KV, hd, ffn, V = shapes[name]
    config = ppsd.TransformerConfig(n, d, H, KV, hd, ffn, V, kv_dtype="fp32", max_ctx=256)
    lm = ppsd.TransformerLM(config, seed=3, deep_scale=0.5, deep_from=1)
    prompt = [int(t) for t in np.random.default_rng(5).integers(0, V, size=70)]
    eng = ppsd.engine_for(lm, ppsd.PipelineConfig(n, 1))
    out = eng.decode_ar(prompt, 4)
    lg = eng.read_logits(1)
    np.save(f"/tmp/lg_{name}_{chunk}.npy", lg)
    print(json.dumps({"chunk": chunk, "tokens": out, "l0": float(lg[0]), "max": float(np.abs(lg).max())}))

if sys.argv[1] == "child":
    child(int(sys.argv[3]))
else:
    name = sys.argv[2]
    for ch in (1, 2, 4, 16):
        subprocess.run([sys.executable, __file__, "child", name, str(ch)])
    base = np.load(f"/tmp/lg_{name}_1.npy")
    for ch in (2, 4, 16):
        o = np.load(f"/tmp/lg_{name}_{ch}.npy")
        print(name, "chunk", ch, "max|diff| vs chunk 1:", float(np.abs(o - base).max()), "bitexact:", bool((o == base).all()))
    from oracle.transformer import ModelShape, TransformerOracle
    shapes = {"mid": (8, 1024, 16, 4, 64, 2816, 4096), "l7b": (2, 4096, 32, 32, 128, 11008, 32000)}
    n, d, H, KV, hd, ffn, V = shapes[name]
    orc = TransformerOracle(ModelShape(n, d, H, KV, hd, ffn, V), seed=3, deep_scale=0.5, deep_from=1, max_ctx=256, threads=16)
    prompt = [int(t) for t in np.random.default_rng(5).integers(0, V, size=70)]
    want = orc.logits_for_prefix(prompt)
    for ch in (1, 16):
        o = np.load(f"/tmp/lg_{name}_{ch}.npy")
        print(name, "chunk", ch, "max|diff| vs oracle:", float(np.abs(o - want).max()), "scale", float(np.abs(want).max()))
