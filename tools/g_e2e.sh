mkdir -p gpurun_out
python tools/diag_e2e.py > gpurun_out/diag_e2e.log 2>&1
VXM_TRACE_HOST=1 python tools/diag_e2e.py > gpurun_out/diag_e2e_trace.log 2>&1
for i in 1 2; do python bench.py --config c5 --steps 10 --warmup 4 --no-cpu-baseline; done > gpurun_out/c5_e2e.log 2>&1
