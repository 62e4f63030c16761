mkdir -p gpurun_out
out=gpurun_out/sanitizer_eig_r2.txt
echo "# compute-sanitizer on tools/sanitize_eig.py (r2 eigensolver + cov_tc)" > $out
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> $out
  timeout 900 compute-sanitizer --tool $tool --print-limit 8 python tools/sanitize_eig.py >> $out 2>&1; echo "rc $?" >> $out
done
