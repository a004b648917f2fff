# round-2: ncu --set full of the cfg5 / cfg4 / cfg2 dominant kernels after the one-IMAD sign flip
mkdir -p gpurun_out/mix
prof() {
  local B="python bench.py --workload $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --graph off"
  timeout 300 $B > gpurun_out/mix/plain_$1.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$3 -s 3 -c 1 \
        -o gpurun_out/mix/prof_$1 $B > gpurun_out/mix/ncu_$1.log 2>&1
  echo "prof $1 rc=$?"
}
prof batch cfg5 '^k_oscprob_batch$'
prof batch_pt cfg4 k_oscprob_batch_pt
prof gl cfg2 k_gl_integrate
# post-process on the box (reports are ~20 MB each)
python tools/sass_mix.py gpurun_out/mix/prof_batch.ncu-rep --points 8e8 > gpurun_out/mix/mix_batch.txt 2>&1
python tools/sass_mix.py gpurun_out/mix/prof_batch_pt.ncu-rep --points 1e8 > gpurun_out/mix/mix_batch_pt.txt 2>&1
python tools/sass_mix.py gpurun_out/mix/prof_gl.ncu-rep --points 1e6 > gpurun_out/mix/mix_gl.txt 2>&1
for n in batch batch_pt gl; do
  ncu -i gpurun_out/mix/prof_$n.ncu-rep --page raw --csv > gpurun_out/mix/raw_$n.csv 2>&1
  ncu -i gpurun_out/mix/prof_$n.ncu-rep --page source --csv --print-source sass > gpurun_out/mix/src_$n.csv 2>&1
done
rm -f gpurun_out/mix/*.ncu-rep
