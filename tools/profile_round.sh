#!/bin/bash
# GPU side: the round's evidence set — every bench line, the default command's launch list,
# and one ncu --set full capture per dominant kernel (each after its own plain run exits 0).
set -u
R=${ROUND:-r01}
mkdir -p gpurun_out/final
if [ -z "${PROF_ONLY:-}" ]; then
for w in cfg5 cfg4 cfg3 cfg2 cfg1 cfg4grid cfg3emu cfg5fit; do
  timeout 400 python bench.py --workload $w > gpurun_out/final/bench_$w.log 2>&1; echo "$w rc=$?"
done
for w in cfg5 cfg4 cfg3 cfg2; do
  timeout 400 python bench.py --workload $w --precision mixed > gpurun_out/final/bench_${w}_mixed.log 2>&1
  echo "$w mixed rc=$?"
done
timeout 300 python bench.py --impl reference > gpurun_out/final/bench_reference.log 2>&1; echo "ref rc=$?"
D="python bench.py --steps 20 --warmup 3"
timeout 400 $D > gpurun_out/final/plain_default.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/final/launches_default.csv $D > gpurun_out/final/ncu_launch.log 2>&1
echo "launches rc=$?"
fi
prof() {  # name workload kernel-regex [extra bench args]; PROFS="a b" limits the set
  case " ${PROFS:-$1} " in *" $1 "*) ;; *) return 0 ;; esac
  local B="python bench.py --workload $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph off ${4:-}"
  timeout 300 $B > gpurun_out/final/plain_$1.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 \
        -o gpurun_out/final/prof_$1 $B > gpurun_out/final/ncu_$1.log 2>&1
  echo "prof $1 rc=$?"
}
prof batch cfg5 '^k_oscprob_batch$'
prof batch_pt cfg4 k_oscprob_batch_pt
prof batch_pt_mixed cfg4 k_oscprob_batch_pt "--precision mixed"
prof eval cfg3 k_oscprob_eval_tma
prof eval_ab cfg3emu k_oscprob_eval_tma
prof gl cfg2 k_gl_integrate
prof scan cfg4grid k_scan_expand
prof scan_setup cfg4grid k_scan_setup
prof batch_mixed cfg5 '^k_oscprob_batch$' "--precision mixed"
