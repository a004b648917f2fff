#!/bin/bash
# GPU side, one call: the round's full evidence set, post-processed on the box so only
# summaries come back (each ncu --set full report is ~20 MB; gpurun returns <= 64 MiB).
#   1. ncu captures (PROF_ONLY) -> install_profiles (ncu_traffic.json updated)
#   2. every bench line (read the updated traffic) + launch list -> install_profiles
#   3. profiles/ copied to gpurun_out/final_prof/, reports deleted except the dominant kernel's
set -u
R=${ROUND:-r01}
mkdir -p gpurun_out/final
PROF_ONLY=1 bash tools/profile_round.sh
python tools/install_profiles.py --round $R --src gpurun_out/final
PROFS=none bash tools/profile_round.sh
python tools/install_profiles.py --round $R --src gpurun_out/final
mkdir -p gpurun_out/final_prof
cp profiles/${R}_* profiles/ncu_traffic.json gpurun_out/final_prof/
find gpurun_out/final -name '*.ncu-rep' ! -name 'prof_batch.ncu-rep' -delete
