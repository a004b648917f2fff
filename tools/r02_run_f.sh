C="python bench.py --workload cfg4grid --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain_f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 2 -o gpurun_out/prof_scan_r02 $C > gpurun_out/ncu_f.log 2>&1
tail -3 gpurun_out/ncu_f.log
