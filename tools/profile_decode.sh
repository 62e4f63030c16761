#!/bin/bash
# ncu evidence for the decode kernel of one bench config (run under gpurun, 1 GPU)
cfg=${1:-llava_b32}
tag=${2:-r1}
mkdir -p gpurun_out
# launch list of the whole bench step (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${cfg}_${tag}.csv \
  python bench.py --config $cfg --steps 2 --warmup 1 --skip-e2e --skip-cpu --no-graph --layers 2 > /dev/null 2>&1
# full capture of one decode launch
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_(fast|gqa)" -s 2 -c 1 \
  -o gpurun_out/prof_decode_${cfg}_${tag} -f \
  python bench.py --config $cfg --steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu --no-graph --layers 1 > gpurun_out/ncu_${cfg}_${tag}.log 2>&1
