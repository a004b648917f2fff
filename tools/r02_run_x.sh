timeout 300 python -m pytest tests -m gpu -x -q -k scan > gpurun_out/x_pytest.log 2>&1; tail -1 gpurun_out/x_pytest.log
for v in base scan_a2_8 scan_a2_12 scan_a2_16 scan_a2_2; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline $L > gpurun_out/x_$v.jsonl 2>&1
done
