mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_sz.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_sz.log
python tools/ab.py 3 c1,c2 head cur 2>&1 | tee gpurun_out/ab16.log
