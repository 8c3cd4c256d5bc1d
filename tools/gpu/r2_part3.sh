mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_partitioned.py -x -q -k bulk > gpurun_out/part3_tests.log 2>&1; echo "part tests rc=$?"; tail -2 gpurun_out/part3_tests.log
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 head default > gpurun_out/part3_ab.log 2>&1; echo "ab rc=$?"; grep median gpurun_out/part3_ab.log
timeout 900 python tools/tools_partition_cost.py 3:0 > gpurun_out/part3_cost.log 2>&1; echo "cost rc=$?"; cat gpurun_out/part3_cost.log | tail -4
PHX_STEP_TIMES=1 timeout 600 python tools/tools_config_roofline.py 3:0 --once > gpurun_out/part3_steps.log 2>&1; grep "step durations" gpurun_out/part3_steps.log | cut -c1-600
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_l2 tools/microbench_l2.cu && timeout 300 /tmp/mb_l2 > gpurun_out/part3_l2.log 2>&1; tail -20 gpurun_out/part3_l2.log
