mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_params_port.py tests/test_gpu_parity.py -x -q -m gpu -k "selection or fixture or full_size or params" > gpurun_out/sel2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/sel2_tests.log
PHX_PROFILE=1 timeout 600 python tools/tools_selection_profile.py > gpurun_out/sel2_prof.log 2>&1; cat gpurun_out/sel2_prof.log | tail -8
