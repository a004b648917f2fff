# round-2: points-across-lanes kernel with order 10 as a constant (fp64 and mixed tier)
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or fit or host" > gpurun_out/pytest_pt3.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pt3.log
for rep in 1 2; do
for v in base pt_noord; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_pt3_cfg4_${v}_$rep.jsonl 2>&1
  timeout 300 python bench.py --workload cfg4 --precision mixed --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_pt3_cfg4mx_${v}_$rep.jsonl 2>&1
done
done
