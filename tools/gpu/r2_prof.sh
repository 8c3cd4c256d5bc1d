mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/p_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c3.csv $CMD > gpurun_out/p_launch.log 2>&1; echo "launch rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_phimv_bulk -c 1 -o gpurun_out/r2_c3_bulk -f python tools/tools_config_roofline.py 3:0 --once > gpurun_out/p_c3full.log 2>&1; echo "c3 full rc=$?"
python tools/tools_config_roofline.py 1:0 4:0 5:2097152 > gpurun_out/p_cfgs.log 2>&1; echo "cfgs rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_phimv -c 1 -o gpurun_out/r2_c1 -f python tools/tools_config_roofline.py 1:0 --once > gpurun_out/p_c1.log 2>&1; echo "c1 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:k_phimv -c 1 --log-file gpurun_out/r2_c5_dram.csv python tools/tools_config_roofline.py 5:2097152 --once > gpurun_out/p_c5.log 2>&1; echo "c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:k_phimv -c 1 --log-file gpurun_out/r2_c4_dram.csv python tools/tools_config_roofline.py 4:0 --once > gpurun_out/p_c4.log 2>&1; echo "c4 rc=$?"
