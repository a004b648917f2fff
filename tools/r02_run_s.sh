timeout 900 python -m pytest tests -m gpu -x -q -k "batch" > gpurun_out/pytest_s.log 2>&1; tail -2 gpurun_out/pytest_s.log
for v in base pt_noshared; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4 --steps 100 --warmup 5 --no-cpu-baseline $L > gpurun_out/s_cfg4_$v.jsonl 2>&1
  timeout 300 python bench.py --workload cfg5 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/s_cfg5_$v.jsonl 2>&1
done
