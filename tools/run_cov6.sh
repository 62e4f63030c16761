mkdir -p gpurun_out
for c in llava_b32 qwen_b32_r32 long_b16; do timeout 300 python tools/time_calib.py $c > gpurun_out/time_calib_cov6_$c.txt 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -k "calibrate or full_size or end_to_end or mode or offline or token or eig or subspace or shard" > gpurun_out/gputest_cov6.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_cov6.log
timeout 600 ncu --set full --clock-control none -k regex:"cov_tc" -c 1 -o gpurun_out/prof_cov6 -f python tools/prof_calib.py llava_b32 > gpurun_out/ncu_cov6.log 2>&1
ncu -i gpurun_out/prof_cov6.ncu-rep --page details --csv > gpurun_out/ncu_cov6_details.csv 2>/dev/null
ncu -i gpurun_out/prof_cov6.ncu-rep --page raw --csv > gpurun_out/ncu_cov6_raw.csv 2>/dev/null
rm -f gpurun_out/prof_cov6.ncu-rep
