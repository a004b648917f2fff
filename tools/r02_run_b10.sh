# round-2: per-point batch kernel with order 10 as a constant; term-loop unroll retest
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or fit or host" > gpurun_out/pytest_b10.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_b10.log
for rep in 1 2; do
for v in base b_noord b_ju1 b_ju3 b_ju4; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg5 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_b10_cfg5_${v}_$rep.jsonl 2>&1
done
done
