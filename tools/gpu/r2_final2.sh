mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f2_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/f2_gputests.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f2_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/f2_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/f2_bench.log | cut -c1-300
