mkdir -p gpurun_out
timeout 1500 python tools/tools_ab_libs.py 3:0 5 2 default c10b2 c12b2 c12 > gpurun_out/cons_ab.log 2>&1; grep "median\|bitwise\|FAIL" gpurun_out/cons_ab.log; grep "c1" gpurun_out/cons_ab.log | head -3 | cut -c1-250
