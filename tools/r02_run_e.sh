python tools/fill_probe.py > gpurun_out/fill_probe.json 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg5_e.jsonl 2>&1
python bench.py --workload cfg4grid --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/scan_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_cfg4grid.csv python bench.py --workload cfg4grid --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_scan.log 2>&1
