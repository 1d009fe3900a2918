#!/bin/bash
# ncu evidence for profiles/: the launch list (per-launch durations) of the C2
# bench command, and one --set full capture per dominant kernel and config.
set -x
mkdir -p gpurun_out
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/launches_c2.log 2>&1
full() {  # name regex skip script args...
  local name=$1 rx=$2 skip=$3; shift 3
  $NCU --set full --import-source on -k regex:$rx --launch-skip $skip --launch-count 1 -f \
    -o gpurun_out/$name "$@" > /dev/null 2>&1
}
full c2_lower k_lower 5 python tools/frames.py c2 7
full c2_integrate k_integrate 5 python tools/frames.py c2 7
full c2_mark k_mark 5 python tools/frames.py c2 7
full c2_rays k_rays 5 python tools/frames.py c2 7
full c2_dilate k_dilate 5 python tools/frames.py c2 7
full c3_integrate k_integrate 4 python tools/frames.py c3 6
full c3_lower k_lower 4 python tools/frames.py c3 6
full c5_lower k_lower 2 python tools/c5_steps.py 3
full c4_lower k_lower 5 python tools/frames.py c4 7
full c1_rays k_rays 5 python tools/frames.py c1 7
full c1_integrate k_integrate 5 python tools/frames.py c1 7
ls -la gpurun_out/*.ncu-rep
