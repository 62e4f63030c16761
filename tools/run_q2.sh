mkdir -p gpurun_out
for c in llava_b32 qwen_b32_r32; do ROTATEK_HJ_SWEEPS=1 timeout 300 python tools/time_calib.py $c > gpurun_out/time_calib_q2_$c.txt 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -k "eig or calibrate or end_to_end or full_size or mode or offline" > gpurun_out/gputest_q2.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_q2.log
