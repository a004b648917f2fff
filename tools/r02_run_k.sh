timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_k.log 2>&1; tail -2 gpurun_out/pytest_gpu_k.log
for v in base sign_on_p base; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  for w in cfg5 cfg4 cfg3; do
    timeout 300 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L >> gpurun_out/k_$w.jsonl 2>&1
  done
  python tools/gl_b2b.py $L --tag $v --cases 100:5,100000:10,1000000:10 >> gpurun_out/k_gl.jsonl 2>&1
done
