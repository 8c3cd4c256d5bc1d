mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_bulk.py tests/test_partitioned.py -x -q -k "bulk" > gpurun_out/early_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/early_tests.log
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 default early0 > gpurun_out/early_ab.log 2>&1; grep "median\|bitwise" gpurun_out/early_ab.log
timeout 900 python tools/tools_ab_libs.py 5:2097152 2 1 default early0 > gpurun_out/early_c5.log 2>&1; grep "median\|bitwise" gpurun_out/early_c5.log
PHX_STEP_TIMES=1 timeout 300 python tools/tools_config_roofline.py 3:0 --once 2>&1 | grep "durations" | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/early_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/early_ref.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['cpu_baseline']['sample'][-200:])"
