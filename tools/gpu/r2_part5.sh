mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_partitioned.py -x -q -k bulk > gpurun_out/part5_tests.log 2>&1; echo "part tests rc=$?"; tail -2 gpurun_out/part5_tests.log
timeout 900 python tools/tools_part_steps.py 3:0 1 2 4 8 > gpurun_out/part5_steps.log 2>&1; echo rc=$?; grep kernel_ms gpurun_out/part5_steps.log; grep "durations" gpurun_out/part5_steps.log | cut -c1-200
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 head default > gpurun_out/part5_ab.log 2>&1; echo "ab rc=$?"; grep median gpurun_out/part5_ab.log
