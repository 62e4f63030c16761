mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "calibrate or select or full_size or end_to_end or mode or offline or token or eig or subspace or shard or smoke" > gpurun_out/gputest_sig.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_sig.log
timeout 300 python -m pytest tests -m "not gpu" -q > gpurun_out/cputest_sig.log 2>&1; echo "rc $?" >> gpurun_out/cputest_sig.log
for c in qwen_b1_r32 llava_b32; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sigma" --csv python tools/prof_calib.py $c > gpurun_out/sig_launches_$c.csv 2>&1
done
