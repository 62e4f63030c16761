# round-2 measurement pass after the eigensolver rewrite (run under gpurun): GPU tests, smoke, bench lines for every
# config, the reference arm, ncu captures (tools/profile_all.sh)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest_r2j.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2j.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2j.txt 2>&1; echo "rc $?" >> gpurun_out/smoke_r2j.txt
timeout 900 python bench.py > gpurun_out/bench_llava_b32_r2j.json 2> gpurun_out/bench_llava_b32_r2j.err
for c in qwen_b32_r32 qwen_b32_r64 joint_b64 long_b16 llava_b8 qwen_b8_r32; do
  timeout 600 python bench.py --config $c --skip-extra > gpurun_out/bench_${c}_r2j.json 2> gpurun_out/bench_${c}_r2j.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_llava_b32_r2j.json 2> gpurun_out/bench_reference_r2j.err
TAG=r2j bash tools/profile_all.sh > gpurun_out/profile_r2j.log 2>&1
