# One GPU pass: the full -m gpu suite, smoke, default bench (C2), C1 bench line,
# and the reference arm.  Logs land in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-600
timeout 600 python bench.py --config c1 > gpurun_out/bench_c1.log 2>&1; echo bench c1 rc=$?; tail -1 gpurun_out/bench_c1.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-400
