mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f1_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/f1_gputests.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/f1_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f1_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/f1_bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/f1_bench.log | cut -c1-600
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f1_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/f1_ref.log | cut -c1-400
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f1_launches.csv $CMD > gpurun_out/f1_ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_phimv_bulk -c 1 -o gpurun_out/f1_c3_bulk -f python tools/tools_config_roofline.py 3:0 --once > gpurun_out/f1_ncu_full.log 2>&1; echo "ncu full rc=$?"
