# cov_tc finalize diagnostics at boost clocks (timing only)
# (the NOSTORE / NOSIGMA switches were removed after this ablation; the script documents it)
mkdir -p gpurun_out
prof() {
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cov_tc" -c 1 --csv python tools/prof_calib.py llava_b32 > gpurun_out/covdiag3_$1.csv 2>&1
}
prof default
for v in "-DCOV_DIAG_NOSTORE:nostore" "-DCOV_DIAG_NOSIGMA:nosigma" "-DCOV_DIAG_NOFIN:nofin" "-DCOV_STAGES=3:s3"; do
  flag=${v%%:*}; tag=${v##*:}
  rm -f build/cov_tc.o
  make all NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $flag" > gpurun_out/covdiag3_build_$tag.log 2>&1
  prof $tag
done
