mkdir -p gpurun_out
for c in llava_b32 qwen_b32_r32 long_b16; do ROTATEK_HJ_SWEEPS=1 timeout 300 python tools/time_calib.py $c > gpurun_out/time_calib_hj3_$c.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_eig.py -q -x > gpurun_out/gputest_hj3.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_hj3.log
timeout 900 python -m pytest tests -m gpu -q -x -k "calibrate or full_size or end_to_end or mode or offline or token" >> gpurun_out/gputest_hj3.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_hj3.log
