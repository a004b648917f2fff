timeout 900 python -m pytest tests -m gpu -x -q -k "batch" > gpurun_out/pytest_v.log 2>&1; tail -2 gpurun_out/pytest_v.log
for p in mixed fp64; do
  timeout 300 python bench.py --workload cfg4 --precision $p --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/v_cfg4_$p.jsonl 2>&1
done
timeout 300 python bench.py --workload cfg5 --precision mixed --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/v_cfg5_mixed.jsonl 2>&1
