mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bulk.py -x -q > gpurun_out/ab1_tests.log 2>&1; echo "bulk tests rc=$?"; tail -2 gpurun_out/ab1_tests.log
timeout 1500 python tools/tools_ab_libs.py 3:0 5 2 head,PHX_BULK_FLAGS=2 default,PHX_BULK_FLAGS=2 default,PHX_BULK_FLAGS=6 c16,PHX_BULK_FLAGS=2 c16,PHX_BULK_FLAGS=6 > gpurun_out/ab1_c3.log 2>&1; echo "ab c3 rc=$?"
timeout 900 python tools/tools_ab_libs.py 5:2097152 2 1 head,PHX_BULK_FLAGS=2 default,PHX_BULK_FLAGS=2 default,PHX_BULK_FLAGS=6 c16,PHX_BULK_FLAGS=6 > gpurun_out/ab1_c5.log 2>&1; echo "ab c5 rc=$?"
