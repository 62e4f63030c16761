timeout 900 python tools/compare_dense.py qwen_b32_r32 long_b16 joint_b64 > gpurun_out/compare_dense2.jsonl 2> gpurun_out/compare_dense2.err
