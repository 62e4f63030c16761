# full GPU suite + default bench after the eigensolver rewrite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_r2i.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2i.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2i.txt 2>&1; echo "rc $?" >> gpurun_out/smoke_r2i.txt
timeout 900 python bench.py > gpurun_out/bench_llava_b32_r2i.json 2> gpurun_out/bench_llava_b32_r2i.err
