mkdir -p gpurun_out
timeout 900 python tools/tools_config_roofline.py 5:0 > gpurun_out/c5full.log 2>&1; echo "rc=$?"; grep '^{' gpurun_out/c5full.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_phimv -c 1 --log-file gpurun_out/r2_c5full_dram.csv python tools/tools_config_roofline.py 5:0 --once > gpurun_out/c5full_ncu.log 2>&1; echo "ncu rc=$?"; grep -v "^==" gpurun_out/r2_c5full_dram.csv | cut -d, -f13-15
timeout 600 python -m pytest tests/test_partitioned.py -q -k multi_device > gpurun_out/c5_md.log 2>&1; tail -2 gpurun_out/c5_md.log
