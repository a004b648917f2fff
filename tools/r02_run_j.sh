# round-2 variant sweep: cfg4 points-across-lanes wave shaping, scan expand block shape, GL split
for v in base pt_s1 pt_s4 pt_b23_s1 pt_b23_s2 pt_b24_s4; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e $L > gpurun_out/j_cfg4_$v.jsonl 2>&1
done
for v in base scan_a5 scan_a2 scan_a3 scan_t64; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  timeout 300 python bench.py --workload cfg4grid --steps 200 --warmup 5 --no-cpu-baseline $L > gpurun_out/j_cfg4grid_$v.jsonl 2>&1
done
C=100000:10,1000000:10
for v in base gl_split_bw4 gl_split_bw2_mb5; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  python tools/gl_b2b.py $L --tag $v --cases $C >> gpurun_out/j_gl_b2b.jsonl 2>&1
done
