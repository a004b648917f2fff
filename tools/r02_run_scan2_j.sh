# round-2: scan stage A GL table staged in shared memory + stage B expand3 (registers, nj points per block)
timeout 600 python -m pytest tests -m gpu -x -q -k "scan or fit" > gpurun_out/pytest_scan_j.log 2>&1; tail -2 gpurun_out/pytest_scan_j.log
for v in base scan_x2 scan_x2_cgl scan_cgl scan_nj4 scan_nj6 scan_nj14 scan_nj16; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_cfg4grid_j_$v.jsonl 2>&1
done
for v in base scan_x2 scan_cgl; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg5fit --steps 20 --warmup 3 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_cfg5fit_j_$v.jsonl 2>&1
done
python tools/scan_probe.py > gpurun_out/scan_probe_j.txt 2>&1
C="python bench.py --workload cfg4grid --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain_j.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg4grid_j.csv $C > gpurun_out/ncu_j.log 2>&1
$C > gpurun_out/plain_j2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 2 -o gpurun_out/prof_scan_j $C > gpurun_out/ncu_j2.log 2>&1
tail -2 gpurun_out/ncu_j2.log
