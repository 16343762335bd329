#!/bin/bash
# One-GPU bench lines for the BASELINE configs beyond the headline (folded
# schedule on one B200): 13B E=20, 70B E=20 and E=10, 7B exit sweep.
#   bash tools/run_configs.sh [outdir]
out=${1:-gpurun_out}
mkdir -p "$out"
run() {
  local tag=$1; shift
  timeout 900 python bench.py "$@" --steps 2 --warmup 1 --cpu-budget 0 --no-toy-rows > "$out/cfg_$tag.json" 2> "$out/cfg_$tag.err"
  python - "$out/cfg_$tag.json" "$tag" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[2], d["value"], d["e2e"]["value"], d.get("ar_tokens_per_s"), round(d["alpha_measured"], 3),
          d["config"]["schedule"], d["step_roofline"]["frac"],
          {k: v.get("tokens_per_s") for k, v in d.get("eesd", {}).items()})
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
}
run 13b_e20 --model 13b --exit 20
run 70b_e20 --model 70b --exit 20
for e in 4 12 16; do run 7b_e$e --model 7b --exit $e; done
