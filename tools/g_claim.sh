mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_esdf.py tests/test_gpu_lower_variants.py tests/test_gpu_bench_parity.py -x -q -k "not c3" > gpurun_out/t_claim.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_claim.log
python tools/ab.py 3 c2,c5,c3 head cur 2>&1 | tee gpurun_out/ab10.log
