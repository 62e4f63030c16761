mkdir -p gpurun_out
for c in llava_b32 qwen_b32_r32 qwen_b32_r64 long_b16; do ROTATEK_HJ_SWEEPS=1 timeout 300 python tools/time_calib.py $c > gpurun_out/time_calib_hj12_$c.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_eig.py -q > gpurun_out/gputest_hj12.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_hj12.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hestenes|refine" -c 2 \
  -o gpurun_out/prof_hj12_llava -f python tools/prof_calib.py llava_b32 > gpurun_out/ncu_hj12.log 2>&1
ncu -i gpurun_out/prof_hj12_llava.ncu-rep --page details --csv > gpurun_out/ncu_hj12_llava_details.csv 2>/dev/null
ncu -i gpurun_out/prof_hj12_llava.ncu-rep --page raw --csv > gpurun_out/ncu_hj12_llava_raw.csv 2>/dev/null
rm -f gpurun_out/prof_hj12_llava.ncu-rep
