# Round-end evidence pass: GPU suite, smoke, every bench line, ncu launch list + captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
bash tools/bench_all.sh
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1; echo profile rc=$?
