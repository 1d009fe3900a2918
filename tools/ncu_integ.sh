# one ncu --set full capture of k_integrate (C3 LiDAR frame 4) with source correlation
mkdir -p gpurun_out
ncu --clock-control none --set full --import-source on -k regex:k_integrate --launch-skip 4 --launch-count 1 -f \
  -o gpurun_out/c3_integ python tools/frames.py c3 6 > gpurun_out/ncu_integ.log 2>&1
echo ncu rc=$?
ls -la gpurun_out/*.ncu-rep
