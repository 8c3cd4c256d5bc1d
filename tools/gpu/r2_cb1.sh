mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "column_blocked or full_size" > gpurun_out/cb1_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/cb1_tests.log
timeout 900 python tools/tools_ab_libs.py 4:0 5 2 head default default,PHX_CB=0 default,PHX_CB_ROWS=524288 default,PHX_CB_ROWS=1398102 > gpurun_out/cb1_ab.log 2>&1; echo "ab rc=$?"; grep -v "^{" gpurun_out/cb1_ab.log | tail -8
PHX_STEP_TIMES=1 timeout 600 python tools/tools_config_roofline.py 4:0 --once > gpurun_out/cb1_steps.log 2>&1; grep "durations\|{" gpurun_out/cb1_steps.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:k_phimv -c 1 --log-file gpurun_out/r2_c4cb_dram.csv python tools/tools_config_roofline.py 4:0 --once > gpurun_out/cb1_ncu.log 2>&1; echo "ncu rc=$?"; grep -v "^==" gpurun_out/r2_c4cb_dram.csv | cut -d, -f13-15
