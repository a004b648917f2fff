timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_l.log 2>&1; tail -2 gpurun_out/pytest_gpu_l.log
python tools/e2e_probe.py > gpurun_out/e2e_probe_l.txt 2>&1
for w in cfg5 cfg4 cfg3 cfg2 cfg1; do
  timeout 300 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/l_$w.jsonl 2>&1
done
GNA_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/l_codepath_n2.jsonl 2> gpurun_out/l_codepath_n2.err; echo n2 rc=$?
