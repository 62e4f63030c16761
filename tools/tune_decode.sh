#!/bin/bash
# usage: tools/tune_decode.sh CONFIG  -- runs the decode bench for each (warps,stages) variant
cfg=${1:-llava_b32}
for v in ${VARIANTS:-default 8,2,16 16,1,32 16,2,16 8,2,32 12,1,32 8,1,64}; do
  if [ "$v" = default ]; then unset ROTATEK_DECODE_CFG; else export ROTATEK_DECODE_CFG=$v; fi
  out=$(timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --skip-full --skip-e2e --skip-cpu 2>/dev/null)
  echo "$cfg $v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["us_per_layer"], d["roofline"]["achieved"], d["roofline"]["frac"], d["clocks"])')"
done
