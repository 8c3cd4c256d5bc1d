mkdir -p gpurun_out
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 default planes > gpurun_out/planes_ab.log 2>&1; echo "ab rc=$?"; grep -v "^{" gpurun_out/planes_ab.log | grep "median\|bitwise"
timeout 900 python tools/tools_ab_libs.py 5:2097152 2 1 default planes > gpurun_out/planes_c5.log 2>&1; grep "median\|bitwise" gpurun_out/planes_c5.log
PHX_LIB=planes PHX_STEP_TIMES=1 timeout 300 python tools/tools_config_roofline.py 3:0 --once 2>&1 | grep "durations" | cut -c1-300
