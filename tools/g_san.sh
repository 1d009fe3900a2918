mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/san_$t.txt 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/san_$t.txt
done
VXM_XR_WIDE=2 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_memcheck_wide.txt 2>&1; echo "wide rc=$?"; tail -3 gpurun_out/san_memcheck_wide.txt
