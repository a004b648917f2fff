# round-2: GPU suite, default bench (cfg5), e2e probe, N=2 code path (gloo ranks on GPU 0)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02_c.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02_c.log
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_cfg5_c.jsonl 2> gpurun_out/bench_cfg5_c.err; tail -c 600 gpurun_out/bench_cfg5_c.err
python tools/e2e_probe.py > gpurun_out/e2e_probe_c.txt 2>&1
GNA_BENCH_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --backend gloo --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/codepath_n2_c.jsonl 2> gpurun_out/codepath_n2_c.err; echo rc=$?; tail -c 1500 gpurun_out/codepath_n2_c.err
