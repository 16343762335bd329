import os, sys, dataclasses
sys.path.insert(0, os.getcwd())
import paper_2509_19368_b200 as ppsd
from paper_2509_19368_b200.decode import Engine
config = dataclasses.replace(ppsd.TransformerConfig.llama2_7b(max_ctx=1024), n_layers=4)
lm = ppsd.TransformerLM(config, seed=0)
cfg = ppsd.PipelineConfig(4, 1)
eng = Engine(lm.model_desc(), lm.weights_struct(), cfg, device=lm.device.index)
nv, ctx = int(sys.argv[1]), int(sys.argv[2])
print(eng.probe_attn(nv, ctx, 5))
