export PYTHONUNBUFFERED=1
timeout 300 python tools/e2e_breakdown.py 2 > gpurun_out/s4b_e2e.log 2>&1; tail -4 gpurun_out/s4b_e2e.log
for v in default al1 al2 al3; do
  if [ $v != default ]; then export HQ_LIB=$PWD/tmp_variants/$v/libhoqri_b200.so; fi
  echo "== $v"
  timeout 300 python tools/pass_time.py 2 2>&1 | tail -1
  timeout 300 python tools/timeline.py 2 5 2>&1 | grep -E "span|k_pass|rowgemm"
done
