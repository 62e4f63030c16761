# cov_tc diagnostics: default, 3 stages, no MMA (timing only; results invalid)
mkdir -p gpurun_out
prof() {  # $1 tag
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed -k regex:"cov_tc" -c 1 --csv python tools/prof_calib.py llava_b32 > gpurun_out/covdiag_$1.csv 2>&1
}
prof default
for v in "-DCOV_STAGES=3:s3" "-DCOV_STAGES=2:s2" "-DCOV_DIAG_NOMMA:nomma"; do
  flag=${v%%:*}; tag=${v##*:}
  rm -f build/cov_tc.o
  make all NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $flag" > gpurun_out/covdiag_build_$tag.log 2>&1
  prof $tag
done
