# round-2: stage A split per pair (k_scan_setup_split) + stage B expand3 variants
timeout 600 python -m pytest tests -m gpu -x -q -k "scan or fit" > gpurun_out/pytest_scan_k.log 2>&1; tail -2 gpurun_out/pytest_scan_k.log
for v in base scan_x2 scan_nosplit scan_nosplit_x2 scan_ju2 scan_ju2_nj14 scan_mb4 scan_mb4_nj14 scan_mb4_ju2 scan_nj14; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_cfg4grid_k_$v.jsonl 2>&1
done
for v in base scan_nosplit scan_x2; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg5fit --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_cfg5fit_k_$v.jsonl 2>&1
done
C="python bench.py --workload cfg4grid --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain_k.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 2 -o gpurun_out/prof_scan_k $C > gpurun_out/ncu_k2.log 2>&1
tail -2 gpurun_out/ncu_k2.log
