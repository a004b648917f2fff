# round-2: overlapped scan (reset -> persistent stage A with per-mass-point counters -> PDL stage B)
timeout 300 python -m pytest tests -m gpu -x -q -k "scan or fit" > gpurun_out/pytest_scan_l.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_scan_l.log
for v in base scan_noov scan_ov2 scan_ov3 scan_ov_mb5 scan_ov_mb6 scan_ov_nopdl; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 120 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_cfg4grid_l_$v.jsonl 2>&1
done
for v in base scan_noov scan_ov2; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 120 python bench.py --workload cfg5fit --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_cfg5fit_l_$v.jsonl 2>&1
done
