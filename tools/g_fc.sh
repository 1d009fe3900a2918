mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_integrate.py tests/test_gpu_frame.py tests/test_gpu_bench_parity.py tests/test_gpu_lower_variants.py tests/test_occupancy.py tests/test_gpu_esdf.py -x -q -m gpu -k "not c3" > gpurun_out/t_fc.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_fc.log
python tools/ab.py 3 c1,c2 head cur 2>&1 | tee gpurun_out/ab14.log
