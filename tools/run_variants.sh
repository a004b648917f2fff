#!/bin/bash
# GPU side: time each tuning variant of the batch kernel on cfg5 and cfg4 (bench.py --lib);
# WORKLOADS and PRECISION (fp64|mixed) from the environment.
for v in "$@"; do
  for w in ${WORKLOADS:-cfg5 cfg4}; do
    timeout 300 python bench.py --workload $w --lib build/variants/$v.so --steps 50 --warmup 5 \
      --no-e2e --no-cpu-baseline --precision ${PRECISION:-fp64} > gpurun_out/var_${v}_$w.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/var_${v}_$w.log').read().strip().splitlines()[-1]); print('$v','$w', round(d['value']/1e9,1), 'G/s', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/var_${v}_$w.log
  done
done
