#!/bin/bash
# ncu evidence for every bench config (run under gpurun, 1 GPU):
#   * the launch list of one bench step (decode + full hot path; cold-cache, serialised:
#     compare SHARES, not absolute times)
#   * one full capture of the decode launch (dram bytes -> profiles/ncu_traffic.json)
#   * full captures of the prefill kernels for llava_b32
tag=${TAG:-r1b}
mkdir -p gpurun_out
for cfg in ${CFGS-llava_b32 qwen_b32_r32 joint_b64 long_b16}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${cfg}_${tag}.csv \
    python bench.py --config $cfg --steps 1 --warmup 1 --skip-e2e --skip-cpu --no-graph --layers 2 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_(fast|gqa|ring)" -s 2 -c 1 \
    -o gpurun_out/prof_decode_${cfg}_${tag} -f \
    python bench.py --config $cfg --steps 1 --warmup 1 --skip-full --skip-e2e --skip-cpu --no-graph --layers 1 > gpurun_out/ncu_${cfg}_${tag}.log 2>&1
  ncu -i gpurun_out/prof_decode_${cfg}_${tag}.ncu-rep --page details --csv > gpurun_out/ncu_decode_${cfg}_${tag}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_decode_${cfg}_${tag}.ncu-rep --page raw --csv > gpurun_out/ncu_decode_${cfg}_${tag}_raw.csv 2>/dev/null
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_decode_${cfg}_${tag}.ncu-rep   # gpurun_out/ must stay < 64 MiB
done
if [ -z "$SKIP_PREFILL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cov_tc|compress_tc|hestenes|refine|select_gather|subspace" -c 7 \
    -o gpurun_out/prof_prefill_llava_b32_${tag} -f \
    python tools/prof_calib.py llava_b32 > gpurun_out/ncu_prefill_${tag}.log 2>&1
  ncu -i gpurun_out/prof_prefill_llava_b32_${tag}.ncu-rep --page details --csv > gpurun_out/ncu_prefill_llava_b32_${tag}_details.csv 2>/dev/null
  ncu -i gpurun_out/prof_prefill_llava_b32_${tag}.ncu-rep --page raw --csv > gpurun_out/ncu_prefill_llava_b32_${tag}_raw.csv 2>/dev/null
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/prof_prefill_llava_b32_${tag}.ncu-rep
fi
