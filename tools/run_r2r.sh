# round-2 closing run: full GPU suite, smoke, default bench line (final code)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_r2r.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2r.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2r.txt 2>&1; echo "rc $?" >> gpurun_out/smoke_r2r.txt
timeout 900 python bench.py > gpurun_out/bench_llava_b32_r2r.json 2> gpurun_out/bench_llava_b32_r2r.err
