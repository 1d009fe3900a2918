mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_integrate.py tests/test_gpu_scale.py tests/test_gpu_bench_parity.py tests/test_gpu_frame.py tests/test_occupancy.py tests/test_gpu_pinned_input.py tests/test_mesh.py tests/test_gpu_shard_esdf.py -x -q -m gpu > gpurun_out/t_rl.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_rl.log
python tools/ab.py 2 c3,c1,c2 base cur 2>&1 | tee gpurun_out/ab_rl.log
