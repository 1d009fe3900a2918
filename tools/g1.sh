set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for i in 1 2 3; do timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_$i.log 2>&1; echo "tests run $i rc=$?"; tail -3 gpurun_out/gpu_tests_$i.log; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -2 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -2 gpurun_out/bench_ref.log
