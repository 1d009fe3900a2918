mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lower_variants.py tests/test_gpu_esdf.py tests/test_gpu_bench_parity.py tests/test_gpu_lower_format.py tests/test_gpu_scale.py tests/test_gpu_frame.py tests/test_replay.py tests/test_gpu_host_lists.py tests/test_occupancy.py -x -q -m gpu > gpurun_out/t_ec.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_ec.log
python tools/ab.py 3 c2,c1 base cur 2>&1 | tee gpurun_out/ab_ec.log
