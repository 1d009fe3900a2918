#!/bin/bash
# One A/B pass on the GPU box (run through gpurun): a GPU test subset, then
# tools/ab.py over library variants built under tools/ab/<name>/ (see ab.py).
#   TESTS="tests/test_gpu_esdf.py ..." CONFIGS=c2,c5 ROUNDS=3 VARIANTS="base cur" bash tools/g_ab.sh
mkdir -p gpurun_out
TESTS=${TESTS:-"tests/test_gpu_lower_variants.py tests/test_gpu_esdf.py tests/test_gpu_bench_parity.py"}
timeout 1500 python -m pytest $TESTS -x -q -m gpu > gpurun_out/t_ab.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_ab.log
python tools/ab.py ${ROUNDS:-3} ${CONFIGS:-c2} ${VARIANTS:-base cur} 2>&1 | tee gpurun_out/ab.log
