mkdir -p gpurun_out
VXM_TRACE_XR=1 VXM_LIB_PATH=$PWD/tools/ab/base/libvoxmap_b200.so python tools/trace_lower.py c2 12 > gpurun_out/trace_ec_base.log 2>&1
VXM_TRACE_XR=1 python tools/trace_lower.py c2 12 > gpurun_out/trace_ec_cur.log 2>&1
