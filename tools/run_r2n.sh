# round-2 measurement pass after the eigensolver rewrite (run under gpurun): GPU tests, smoke, bench lines for every
# config, the reference arm, ncu captures (tools/profile_all.sh)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest_r2n.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest_r2n.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2n.txt 2>&1; echo "rc $?" >> gpurun_out/smoke_r2n.txt
timeout 900 python bench.py > gpurun_out/bench_llava_b32_r2n.json 2> gpurun_out/bench_llava_b32_r2n.err
for c in qwen_b32_r32 qwen_b32_r64 joint_b64 long_b16 llava_b8 qwen_b8_r32; do
  timeout 600 python bench.py --config $c --skip-extra > gpurun_out/bench_${c}_r2n.json 2> gpurun_out/bench_${c}_r2n.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference_llava_b32_r2n.json 2> gpurun_out/bench_reference_r2n.err
TAG=r2n bash tools/profile_all.sh > gpurun_out/profile_r2n.log 2>&1
# per-kernel prefill latencies at small U (one matrix per SM): qwen_b32 (128 units), qwen_b8 (32), qwen_b1 (4)
for c in qwen_b32_r32 qwen_b8_r32 qwen_b1_r32; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cov_tc|hestenes|refine|select|sigma" --csv \
    python tools/prof_calib.py $c > gpurun_out/prefill_launches_${c}_r2n.csv 2>&1
done
