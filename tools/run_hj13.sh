mkdir -p gpurun_out
for c in llava_b32 qwen_b32_r32 long_b16; do ROTATEK_HJ_SWEEPS=1 timeout 300 python tools/time_calib.py $c > gpurun_out/time_calib_hj13_$c.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_eig.py -q > gpurun_out/gputest_hj13.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_hj13.log
for c in llava_b32 qwen_b1_r32; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"hestenes" --csv python tools/prof_calib.py $c > gpurun_out/hj13_$c.csv 2>&1
done
