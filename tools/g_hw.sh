mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lower_variants.py tests/test_gpu_esdf.py tests/test_gpu_bench_parity.py tests/test_gpu_lower_format.py tests/test_gpu_scale.py tests/test_gpu_frame.py -x -q -m gpu > gpurun_out/t_hw.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_hw.log
python tools/ab.py 2 c2,c3,c4,c5 base cur 2>&1 | tee gpurun_out/ab_hw.log
