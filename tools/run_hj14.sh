mkdir -p gpurun_out
for c in llava_b32 qwen_b32_r32 long_b16 qwen_b8_r32; do ROTATEK_HJ_SWEEPS=1 timeout 300 python tools/time_calib.py $c > gpurun_out/time_calib_hj14_$c.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_eig.py tests/test_gpu_parity.py -q -k "eig or calibrate or end_to_end or full_size or nonfinite" > gpurun_out/gputest_hj14.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_hj14.log
for c in qwen_b1_r32 qwen_b32_r32 llava_b32; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hestenes" --csv python tools/prof_calib.py $c > gpurun_out/hj14_$c.csv 2>&1
done
