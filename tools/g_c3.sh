mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_scale.py tests/test_gpu_integrate.py tests/test_occupancy.py tests/test_gpu_frame.py -x -q -m gpu > gpurun_out/t_c3.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/t_c3.log
python tools/ab.py 2 c3 c3a cur 2>&1 | tee gpurun_out/ab7.log
