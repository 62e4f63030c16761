set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2c.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2c.txt 2>&1; echo "rc $?" >> gpurun_out/smoke_r2c.txt
timeout 900 python bench.py > gpurun_out/bench_llava_b32_r2c.json 2> gpurun_out/bench_llava_b32_r2c.err
for c in qwen_b32_r32 qwen_b32_r64 joint_b64 long_b16 llava_b8 qwen_b8_r32; do
  timeout 600 python bench.py --config $c --skip-extra > gpurun_out/bench_${c}_r2c.json 2> gpurun_out/bench_${c}_r2c.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_llava_b32_r2c.json 2> gpurun_out/bench_reference_r2c.err
