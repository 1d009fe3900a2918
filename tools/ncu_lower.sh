# one ncu --set full capture of k_lower (C2 frame 5) with source correlation
mkdir -p gpurun_out
ncu --clock-control none --set full --import-source on -k regex:k_lower --launch-skip 5 --launch-count 1 -f \
  -o gpurun_out/c2_lower_cl python tools/frames.py c2 7 > gpurun_out/ncu_lower.log 2>&1
echo ncu rc=$?
ls -la gpurun_out/*.ncu-rep
