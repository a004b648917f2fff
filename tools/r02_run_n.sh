timeout 600 python -m pytest tests -m gpu -x -q -k "scan" > gpurun_out/pytest_scan_n.log 2>&1; tail -2 gpurun_out/pytest_scan_n.log
for v in base scan_cs4 scan_cs2 scan_nocl; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline $L > gpurun_out/n_cfg4grid_$v.jsonl 2>&1
done
