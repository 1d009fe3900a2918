mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_esdf.py tests/test_gpu_lower_variants.py tests/test_gpu_bench_parity.py -x -q -m gpu -k "not c3" > gpurun_out/t_tr.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_tr.log
VXM_TRACE_XR=1 python tools/trace_lower.py c2 4 > gpurun_out/trace_tr.log 2>&1; echo "trace rc=$?"; grep -c 'round ends' gpurun_out/trace_tr.log
python tools/ab.py 3 c2,c5 tr cur 2>&1 | tee gpurun_out/ab18.log
