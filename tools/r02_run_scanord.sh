# round-2: scan stage A with order 10 as a constant (after the one-IMAD sign flip)
timeout 600 python -m pytest tests -m gpu -x -q -k "scan or fit" > gpurun_out/pytest_scanord.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_scanord.log
for rep in 1 2; do
for v in base scan_noord scan_ord_mb6 scan_ord_mb8; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 120 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_scanord_cfg4grid_${v}_$rep.jsonl 2>&1
  timeout 120 python bench.py --workload cfg5fit --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_scanord_cfg5fit_${v}_$rep.jsonl 2>&1
done
done
