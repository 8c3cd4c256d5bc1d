mkdir -p gpurun_out
timeout 900 python tools/tools_ab_libs.py 3:0 5 2 default gb4 > gpurun_out/gb4_ab.log 2>&1; grep "median\|bitwise" gpurun_out/gb4_ab.log
timeout 900 python tools/tools_ab_libs.py 5:2097152 2 1 default gb4 > gpurun_out/gb4_c5.log 2>&1; grep "median\|bitwise" gpurun_out/gb4_c5.log
