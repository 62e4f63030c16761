mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "compress or end_to_end or full_size or token or offline or mode" > gpurun_out/gputest_cmp.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_cmp.log
for c in llava_b32 qwen_b32_r64; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"compress_tc" --csv python tools/prof_calib.py $c > gpurun_out/cmp_launches_$c.csv 2>&1
done
