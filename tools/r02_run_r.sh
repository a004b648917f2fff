for v in base pt_staged pt_staged_mb16 pt_staged_mb20 pt_mb20 pt_mb16 pt_mb12 pt_n10_mb16 pt_n10_mb12; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/r_cfg4_$v.jsonl 2>&1
done
