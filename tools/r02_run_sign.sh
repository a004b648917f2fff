# round-2: sign flip by parity as one IMAD (GNA_SIGN_IMAD) vs shift + XOR (variant sign_lop)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_sign.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_sign.log
for rep in 1 2; do
for v in base sign_lop; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  for w in cfg5 cfg4 cfg3emu cfg5fit cfg2; do
    timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_sign_${w}_${v}_$rep.jsonl 2>&1
  done
  python tools/gl_b2b.py ${L:+--lib build/variants/$v.so} --tag $v > gpurun_out/gl_b2b_sign_${v}_$rep.jsonl 2>&1
done
done
