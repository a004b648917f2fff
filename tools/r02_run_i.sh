timeout 600 python -m pytest tests -m gpu -x -q -k "scan" > gpurun_out/pytest_scan_i.log 2>&1; tail -2 gpurun_out/pytest_scan_i.log
for v in base scan_noexp2; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline $L > gpurun_out/bench_cfg4grid_i_$v.jsonl 2>&1
done
C="python bench.py --workload cfg4grid --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain_i.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg4grid_i.csv $C > gpurun_out/ncu_i.log 2>&1
