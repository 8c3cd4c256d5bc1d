mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_partitioned.py tests/test_bulk.py -x -q > gpurun_out/part1_tests.log 2>&1; echo "part tests rc=$?"; tail -15 gpurun_out/part1_tests.log
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 head default > gpurun_out/part1_ab.log 2>&1; echo "ab rc=$?"; grep median gpurun_out/part1_ab.log
timeout 900 python tools/tools_partition_cost.py 3:0 > gpurun_out/part1_cost.log 2>&1; echo "cost rc=$?"; cat gpurun_out/part1_cost.log | tail -5
