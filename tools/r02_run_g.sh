timeout 600 python -m pytest tests -m gpu -x -q -k "scan" > gpurun_out/pytest_scan_g.log 2>&1; tail -3 gpurun_out/pytest_scan_g.log
for v in base scan_unfused scan_b64_c4 scan_c2 scan_c8 scan_c4_mb3; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4grid --steps 100 --warmup 5 --no-cpu-baseline $L > gpurun_out/bench_cfg4grid_g_$v.jsonl 2>&1
done
