# round-2 GL / elementwise launch-floor study (back-to-back launches, tools/gl_b2b.py)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02_b.log 2>&1; tail -3 gpurun_out/pytest_gpu_r02_b.log
C=100:5,1000:10,10000:10,100000:10,1000000:10,10000000:10
for v in base nopdl_single nopdl_single_nosplit gl_nosplit gl_split_bw2; do
  if [ $v = base ]; then L=""; else L="--lib build/variants/$v.so"; fi
  python tools/gl_b2b.py $L --tag $v --cases $C >> gpurun_out/gl_b2b_r02b.jsonl 2>&1
  python tools/gl_b2b.py $L --tag $v --mode eval --cases 1000:1,100000:1,10000000:1 >> gpurun_out/gl_b2b_r02b.jsonl 2>&1
  python tools/gl_b2b.py $L --tag $v --mode mixed --cases 100000:10 >> gpurun_out/gl_b2b_r02b.jsonl 2>&1
done
python tools/gl_b2b.py --tag base_rep --cases $C >> gpurun_out/gl_b2b_r02b.jsonl 2>&1
