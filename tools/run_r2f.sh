# round-2 re-entry validation (run under gpurun): GPU tests, bench line, calibrate timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_r2f.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2f.log
timeout 600 python bench.py > gpurun_out/bench_llava_b32_r2f.json 2> gpurun_out/bench_llava_b32_r2f.err
timeout 300 python tools/time_calib.py llava_b32 > gpurun_out/time_calib_r2f.txt 2>&1
