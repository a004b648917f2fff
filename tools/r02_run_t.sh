for v in base pt_n10 pt_n10_mb20 pt_s1_sh pt_s4_sh base; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/t_cfg4_$v.jsonl 2>&1
done
