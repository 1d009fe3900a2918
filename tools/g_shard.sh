mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard_esdf.py tests/test_gpu_dist_esdf.py -x -q > gpurun_out/t_shard.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_shard.log
for v in head cur; do
  if [ $v = head ]; then export VXM_LIB_PATH=$PWD/tools/ab/head/libvoxmap_b200.so; else unset VXM_LIB_PATH; fi
  for r in 1 2; do echo "$v"; python tools/shard_time.py 256 2 2>&1 | tail -3; done
done
