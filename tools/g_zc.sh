mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_zero_copy.py tests/test_gpu_integrate.py tests/test_gpu_frame.py tests/test_gpu_esdf.py tests/test_gpu_bench_parity.py tests/test_replay.py tests/test_gpu_lidar_angles.py tests/test_abi.py -x -q -m gpu > gpurun_out/t_zc.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_zc.log
python tools/diag_e2e.py > gpurun_out/diag_e2e_zc.log 2>&1; tail -1 gpurun_out/diag_e2e_zc.log
python tools/ab.py 2 c1,c2,c3 base cur cur:VXM_NO_ZERO_COPY=1 2>&1 | tee gpurun_out/ab_zc.log
