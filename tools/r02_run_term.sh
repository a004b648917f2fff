# round-2: single-point kernels with the term loop unrolled (GNA_PROB_TERM_UNROLL)
for v in base term_unroll3 term_unroll3_splitmb2; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  python tools/gl_b2b.py $L --tag $v > gpurun_out/gl_b2b_term_${v}.jsonl 2>&1
  python tools/gl_b2b.py $L --tag $v --mode eval --cases 1000:1,100000:1,10000000:1 >> gpurun_out/gl_b2b_term_${v}.jsonl 2>&1
  timeout 300 python bench.py --workload cfg3 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_term_cfg3_${v}.jsonl 2>&1
  timeout 300 python bench.py --workload cfg2 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/bench_term_cfg2_${v}.jsonl 2>&1
done
