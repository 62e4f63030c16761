# round-2 closing run: full GPU suite, smoke, default bench line (final code)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_r2o.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2o.txt 2>&1; echo "rc $?" >> gpurun_out/smoke_r2o.txt
timeout 900 python bench.py > gpurun_out/bench_llava_b32_r2o.json 2> gpurun_out/bench_llava_b32_r2o.err
