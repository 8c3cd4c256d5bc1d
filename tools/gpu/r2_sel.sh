mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_params_port.py tests/test_gpu_parity.py tests/test_partitioned.py tests/test_phi_port.py -x -q -m gpu > gpurun_out/sel_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sel_tests.log
PHX_PROFILE=1 timeout 600 python tools/tools_selection_profile.py > gpurun_out/sel_prof.log 2>&1; cat gpurun_out/sel_prof.log | tail -8
