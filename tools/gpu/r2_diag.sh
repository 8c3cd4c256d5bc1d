mkdir -p gpurun_out
for v in default diag1 diag2 diag3; do
  if [ $v = default ]; then unset PHX_LIB; else export PHX_LIB=$v; fi
  echo "== $v"; PHX_STEP_TIMES=1 timeout 300 python tools/tools_config_roofline.py 3:0 --once 2>&1 | grep "durations\|kernel_ms" | cut -c1-330
done > gpurun_out/diag.log 2>&1
cat gpurun_out/diag.log
