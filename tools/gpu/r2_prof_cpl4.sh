mkdir -p gpurun_out
timeout 300 python tools/tools_part_steps.py 3:0 1 > gpurun_out/steps_cpl4.log 2>&1; echo "steps rc=$?"
PHX_LIB=cpl2 timeout 300 python tools/tools_part_steps.py 3:0 1 > gpurun_out/steps_cpl2.log 2>&1; echo "steps2 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_phimv_bulk -c 1 -o gpurun_out/r2_c3_cpl4 -f python tools/tools_config_roofline.py 3:0 --once > gpurun_out/p_c3cpl4.log 2>&1; echo "c3 full rc=$?"
