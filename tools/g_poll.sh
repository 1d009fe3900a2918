mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_poll.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_poll.log
python tools/ab.py 2 c1,c2,c3 base cur cur:VXM_SYNC_POLL=0 2>&1 | tee gpurun_out/ab_poll.log
