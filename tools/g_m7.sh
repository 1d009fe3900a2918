mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_esdf.py tests/test_gpu_bench_parity.py tests/test_gpu_frame.py tests/test_gpu_scale.py tests/test_occupancy.py tests/test_replay.py -x -q -m gpu > gpurun_out/t_m7.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_m7.log
python tools/ab.py 2 c2,c3,c5 base cur 2>&1 | tee gpurun_out/ab_m7.log
