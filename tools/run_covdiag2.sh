# cov_tc diagnostics at boost clocks: default, no MMA, no fp64 drain, no finalize (timing only)
mkdir -p gpurun_out
prof() {
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"cov_tc" -c 1 --csv python tools/prof_calib.py llava_b32 > gpurun_out/covdiag2_$1.csv 2>&1
}
prof default
for v in "-DCOV_DIAG_NOMMA:nomma" "-DCOV_DIAG_NODRAIN:nodrain" "-DCOV_DIAG_NOFIN:nofin" "-DCOV_DIAG_NOFIN -DCOV_DIAG_NODRAIN:nofin_nodrain" "-DCOV_DIAG_NOFIN -DCOV_DIAG_NODRAIN -DCOV_DIAG_NOMMA:none"; do
  flag=${v%%:*}; tag=${v##*:}
  rm -f build/cov_tc.o
  make all NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $flag" > gpurun_out/covdiag2_build_$tag.log 2>&1
  prof $tag
done
