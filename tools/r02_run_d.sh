# round-2: host pipeline (3 streams) + scan expand variants
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02_d.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02_d.log
python tools/e2e_probe.py > gpurun_out/e2e_probe_d.txt 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg5_d.jsonl 2>&1
python bench.py --workload cfg3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_d.jsonl 2>&1
python bench.py --workload cfg2 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg2_d.jsonl 2>&1
python bench.py --workload cfg4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_cfg4_d.jsonl 2>&1
for v in base scan_a8 scan_a16 scan_a8_t256 scan_a16_t256; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  python bench.py --workload cfg4grid --steps 100 --warmup 5 --no-cpu-baseline $L > gpurun_out/bench_cfg4grid_$v.jsonl 2>&1
done
