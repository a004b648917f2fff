mkdir -p gpurun_out/final
timeout 400 python bench.py --workload cfg4 > gpurun_out/final/bench_cfg4.log 2>&1; echo "cfg4 rc=$?"
PROFS="batch_pt" PROF_ONLY=1 bash tools/profile_round.sh
