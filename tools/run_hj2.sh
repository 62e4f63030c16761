mkdir -p gpurun_out
for c in llava_b32 qwen_b32_r32; do ROTATEK_HJ_SWEEPS=1 timeout 300 python tools/time_calib.py $c > gpurun_out/time_calib_hj2_$c.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hestenes|refine_smem" -c 2 \
  -o gpurun_out/prof_hj_llava -f python tools/prof_calib.py llava_b32 > gpurun_out/ncu_hj.log 2>&1
ncu -i gpurun_out/prof_hj_llava.ncu-rep --page details --csv > gpurun_out/ncu_hj_llava_details.csv 2>/dev/null
ncu -i gpurun_out/prof_hj_llava.ncu-rep --page raw --csv > gpurun_out/ncu_hj_llava_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_hj_llava.ncu-rep --page source --csv -k regex:hestenes > gpurun_out/ncu_hj_llava_source.csv 2>/dev/null
