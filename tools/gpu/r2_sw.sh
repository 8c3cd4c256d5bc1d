mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_bulk.py tests/test_partitioned.py tests/test_gpu_parity.py -x -q -k "bulk or full_size or stablenorm or production" > gpurun_out/sw_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/sw_tests.log
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 default swall > gpurun_out/sw_ab.log 2>&1; grep "median\|bitwise" gpurun_out/sw_ab.log
PHX_STEP_TIMES=1 timeout 300 python tools/tools_config_roofline.py 3:0 --once 2>&1 | grep "durations" | cut -c1-300
