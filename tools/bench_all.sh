#!/bin/bash
# Final bench lines of every config (+ the reference arm on C2) into gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-160
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_c2.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_c2.log | cut -c1-200
