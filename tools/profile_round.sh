#!/bin/bash
# ncu evidence for profiles/: launch lists (per-launch durations) of the C2
# bench command, and one --set full capture per dominant kernel and config.
set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c2.log 2>&1
$NCU --set full --import-source on -k regex:k_lower3 --launch-skip 5 --launch-count 1 -f -o gpurun_out/c2_lower python tools/frames.py c2 7 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:k_integrate --launch-skip 5 --launch-count 1 -f -o gpurun_out/c2_integrate python tools/frames.py c2 7 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:k_mark --launch-skip 5 --launch-count 1 -f -o gpurun_out/c2_mark python tools/frames.py c2 7 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:k_lower3 --launch-skip 2 --launch-count 1 -f -o gpurun_out/c5_lower python tools/c5_steps.py 3 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:k_integrate --launch-skip 4 --launch-count 1 -f -o gpurun_out/c3_integrate python tools/frames.py c3 6 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:k_lower3 --launch-skip 4 --launch-count 1 -f -o gpurun_out/c3_lower python tools/frames.py c3 6 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
