timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 400 python bench.py > gpurun_out/bench_llava_b32_r1e.json 2> gpurun_out/bench_llava_b32_r1e.err
for c in qwen_b32_r32 joint_b64 long_b16 qwen_b32_r64 llava_b8 qwen_b8_r32; do timeout 400 python bench.py --config $c --skip-e2e --skip-cpu > gpurun_out/bench_${c}_r1e.json 2>gpurun_out/bench_${c}_r1e.err; done
CFGS="llava_b32" TAG=r1e bash tools/profile_all.sh > gpurun_out/profile_all.log 2>&1
timeout 600 python __graft_entry__.py 2>&1 | tail -3 > gpurun_out/smoke_r1e.txt || true
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1e.txt 2>&1
