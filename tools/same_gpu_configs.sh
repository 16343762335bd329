#!/bin/bash
# BASELINE's multi-GPU configurations (13B E=20 on 2 ranks, 70B E=20 on 4,
# 70B E=10 on 8) run through bench.py's multi-rank path with every rank on
# cuda:0 (PPSD_BENCH_SAME_GPU=1: a correctness run of the rank split, peer
# stores and per-rank fold on one device; its tokens/s is NOT a multi-GPU
# number), each against the 1-GPU engine of the same config: the token
# digests, ticks, accepts and rejects must be equal.
#   bash tools/same_gpu_configs.sh [outdir]
out=${1:-gpurun_out/same_gpu}
mkdir -p "$out"
cmp() {
  python - "$out/n1_$1.json" "$out/n$2_$1.json" "$1" "$2" <<'PY'
import json, sys
try:
    a, b = (json.loads(open(p).read().strip().splitlines()[-1]) for p in sys.argv[1:3])
    keys = ("tokens_digest", "ticks", "accepts", "rejects")
    same = all(a.get(k) == b.get(k) for k in keys)
    print(json.dumps({"config": sys.argv[3], "ranks": int(sys.argv[4]), "identical": same,
                      "n1": {k: a.get(k) for k in keys}, "same_gpu": {k: b.get(k) for k in keys},
                      "n1_tok_s": a["value"], "same_gpu_tok_s": b["value"],
                      "transport": b["config"].get("transport")}))
except Exception as e:  # noqa: BLE001
    print(json.dumps({"config": sys.argv[3], "ranks": int(sys.argv[4]), "failed": str(e)}))
PY
}
run() {  # tag ranks model exit
  local tag=$1 n=$2 m=$3 e=$4
  timeout 900 python bench.py --model "$m" --exit "$e" --steps 1 --warmup 1 --cpu-budget 0 --no-toy-rows \
    > "$out/n1_$tag.json" 2> "$out/n1_$tag.err"
  PPSD_BENCH_SAME_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" \
    --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus "$n" --model "$m" --exit "$e" \
    --steps 1 --warmup 1 > "$out/n${n}_$tag.json" 2> "$out/n${n}_$tag.err"
  cmp "$tag" "$n" | tee -a "$out/summary.jsonl"
}
run 13b_e20 2 13b 20
run 70b_e20 4 70b 20
run 70b_e10 8 70b 10
