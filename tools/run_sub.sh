mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"subspace_tc" -c 1 \
  -o gpurun_out/prof_sub -f python tools/prof_calib.py llava_b32 > gpurun_out/ncu_sub.log 2>&1
ncu -i gpurun_out/prof_sub.ncu-rep --page source --csv --print-source sass > gpurun_out/sub_sass.csv 2>&1
ncu -i gpurun_out/prof_sub.ncu-rep --page details --csv > gpurun_out/sub_details.csv 2>&1
ncu -i gpurun_out/prof_sub.ncu-rep --page source --csv --print-source cuda > gpurun_out/sub_cuda.csv 2>&1
rm -f gpurun_out/prof_sub.ncu-rep
