mkdir -p gpurun_out
PHX_LIB=probe PHX_STEP_TIMES=1 timeout 300 python tools/tools_config_roofline.py 3:0 --once 2>&1 | grep "probe\|kernel_ms" | cut -c1-400
PHX_LIB=probe PHX_STEP_TIMES=1 timeout 300 python tools/tools_config_roofline.py 5:2097152 --once 2>&1 | grep "probe\|kernel_ms" | cut -c1-400
