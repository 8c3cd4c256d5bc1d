mkdir -p gpurun_out
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 default pf > gpurun_out/pf_ab.log 2>&1; grep "median\|bitwise" gpurun_out/pf_ab.log
PHX_LIB=pf PHX_STEP_TIMES=1 timeout 300 python tools/tools_config_roofline.py 3:0 --once 2>&1 | grep "durations" | cut -c1-300
