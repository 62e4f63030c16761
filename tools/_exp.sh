timeout 400 python bench.py > gpurun_out/bench_llava_b32_r1d.json 2> gpurun_out/bench_llava_b32_r1d.err
for c in qwen_b32_r32 joint_b64 long_b16 qwen_b32_r64; do timeout 400 python bench.py --config $c --skip-e2e --skip-cpu > gpurun_out/bench_${c}_r1d.json 2>gpurun_out/bench_${c}_r1d.err; done
TAG=r1d bash tools/profile_all.sh > gpurun_out/profile_all.log 2>&1
du -sh gpurun_out
