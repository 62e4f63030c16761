#!/bin/bash
# usage: tools/tune_gqa.sh CONFIG -- decode bench for each GQA ring variant (tile,stages)
cfg=${1:-qwen_b32_r32}
for v in ${VARIANTS:-default 32,2 64,2}; do
  if [ "$v" = default ]; then unset ROTATEK_GQA_CFG; else export ROTATEK_GQA_CFG=$v; fi
  out=$(timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --skip-full --skip-e2e --skip-cpu 2>/dev/null)
  echo "$cfg $v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_layer"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done
