# source-level stall sampling of the lone-CTA prefill kernels (qwen_b1: 4 units)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hestenes|select_gather" -c 2 \
  -o gpurun_out/prof_lat -f python tools/prof_calib.py qwen_b1_r32 > gpurun_out/ncu_lat.log 2>&1
ncu -i gpurun_out/prof_lat.ncu-rep --page source --csv --print-source sass -k regex:hestenes > gpurun_out/lat_hestenes_sass.csv 2>&1
ncu -i gpurun_out/prof_lat.ncu-rep --page source --csv --print-source sass -k regex:select_gather > gpurun_out/lat_select_sass.csv 2>&1
ncu -i gpurun_out/prof_lat.ncu-rep --page details --csv > gpurun_out/lat_details.csv 2>&1
rm -f gpurun_out/prof_lat.ncu-rep
