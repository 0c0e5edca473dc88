#!/bin/bash
# Short-chain (small-job) profile: full ncu captures of the sweep of BASELINE C5 n = 16 and
# C2, with the per-SASS-line source page, plus the small-job timing table.
# usage: gpurun --timeout 900 -- 'bash tools/gpu_short.sh TAG'
TAG=${1:-s1}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python tools/small_jobs.py > gpurun_out/small_jobs_$TAG.jsonl 2> gpurun_out/small_jobs_$TAG.err
for pt in c5_16 c2; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 \
    -o gpurun_out/prof_${pt}_$TAG python tools/small_jobs.py --only $pt --reps 1 > gpurun_out/ncu_${pt}_$TAG.log 2>&1
  if [ -f gpurun_out/prof_${pt}_$TAG.ncu-rep ]; then
    ncu -i gpurun_out/prof_${pt}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${pt}_${TAG}_raw.csv 2>/dev/null
    ncu -i gpurun_out/prof_${pt}_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${pt}_${TAG}_src.csv 2>/dev/null
  fi
done
rm -f gpurun_out/*.ncu-rep
echo done
