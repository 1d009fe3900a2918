mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_lower_variants.py tests/test_gpu_esdf.py tests/test_gpu_bench_parity.py tests/test_gpu_frame.py -x -q -m gpu > gpurun_out/t_ec2.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ec2.log
VXM_TRACE_XR=1 python tools/trace_lower.py c2 12 > gpurun_out/trace_ec_cur2.log 2>&1
python tools/ab.py 3 c2 base cur 2>&1 | tee gpurun_out/ab_ec2.log
