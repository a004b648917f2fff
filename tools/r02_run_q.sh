B="python bench.py --workload cfg4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph off"
timeout 300 $B > gpurun_out/plain_q.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_oscprob_batch_pt -s 3 -c 1 -o gpurun_out/prof_pt_r02 $B > gpurun_out/ncu_q.log 2>&1
echo rc=$?
