mkdir -p gpurun_out
timeout 900 python tools/tools_part_steps.py 3:0 1 2 8 > gpurun_out/part4_steps.log 2>&1; echo rc=$?; cut -c1-400 gpurun_out/part4_steps.log
