set -x
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -x -q > gpurun_out/final/gputests.log 2>&1; tail -3 gpurun_out/final/gputests.log
python bench.py > gpurun_out/final/bench_c3.jsonl 2> gpurun_out/final/bench_c3.err
python bench.py --impl reference > gpurun_out/final/bench_ref.jsonl 2> gpurun_out/final/bench_ref.err
python tools/tools_config_roofline.py 2:0 4:0 1:0 5:2097152 > gpurun_out/final/config_roofline.jsonl 2> gpurun_out/final/config_roofline.err
python tools/tools_config_roofline.py --once 5:0 >> gpurun_out/final/config_roofline.jsonl 2>> gpurun_out/final/config_roofline.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/c3_launches.csv $CMD > gpurun_out/final/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_phimv_bulk -s 1 -c 1 -o gpurun_out/final/prof_c3 $CMD > gpurun_out/final/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_phimv_bulk -s 1 -c 1 --csv --log-file gpurun_out/final/c5_metrics.csv python tools/tools_config_roofline.py 5:2097152 > gpurun_out/final/ncu_c5.log 2>&1
ls -la gpurun_out/final
