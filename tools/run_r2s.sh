# final per-config bench lines on the final code
mkdir -p gpurun_out
for c in qwen_b32_r32 qwen_b32_r64 joint_b64 long_b16 llava_b8 qwen_b8_r32; do
  timeout 600 python bench.py --config $c --skip-extra > gpurun_out/bench_${c}_r2s.json 2> gpurun_out/bench_${c}_r2s.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_llava_b32_r2s.json 2> gpurun_out/bench_reference_r2s.err
