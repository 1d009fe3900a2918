mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_host_lists.py tests/test_gpu_esdf.py tests/test_abi.py tests/test_gpu_bench_parity.py tests/test_gpu_shard_esdf.py tests/test_snapshot.py tests/test_mesh.py -x -q -m gpu > gpurun_out/t_hl.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_hl.log
python tools/ab.py 3 c5 base cur 2>&1 | tee gpurun_out/ab_hl.log
python tools/ab.py 1 c2 base cur 2>&1 | tee -a gpurun_out/ab_hl.log
