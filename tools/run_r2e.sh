# round-2 final measurement pass (run under gpurun): GPU tests, smoke, bench lines for every
# config, the reference arm, ncu captures (tools/profile_all.sh)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest_r2e.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2e.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2e.txt 2>&1; echo "rc $?" >> gpurun_out/smoke_r2e.txt
timeout 900 python bench.py > gpurun_out/bench_llava_b32_r2e.json 2> gpurun_out/bench_llava_b32_r2e.err
for c in qwen_b32_r32 qwen_b32_r64 joint_b64 long_b16 llava_b8 qwen_b8_r32; do
  timeout 600 python bench.py --config $c --skip-extra > gpurun_out/bench_${c}_r2e.json 2> gpurun_out/bench_${c}_r2e.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_llava_b32_r2e.json 2> gpurun_out/bench_reference_r2e.err
TAG=r2e bash tools/profile_all.sh > gpurun_out/profile_r2e.log 2>&1
