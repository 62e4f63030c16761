mkdir -p gpurun_out
TD_KERNEL=3 timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode_ring -s 6 -c 1 -o gpurun_out/prof_ring -f python tools/time_decode.py 128,7,4096,128,32 > gpurun_out/ncu_ring.log 2>&1
ncu -i gpurun_out/prof_ring.ncu-rep --page source --csv > gpurun_out/ncu_ring_source.csv 2>/dev/null
ncu -i gpurun_out/prof_ring.ncu-rep --page details --csv > gpurun_out/ncu_ring_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
