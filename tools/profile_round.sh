#!/bin/bash
# Profiling call for the round's profiles/: launch list of the bench command, full ncu captures
# of the joint sweep (config 4) and the gate build, and the microbenchmarks.
TAG=${1:-r1}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 \
  -o gpurun_out/prof_sweep_$TAG python tools/profile_sweep.py > gpurun_out/ncu_sweep_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gate_build -c 1 \
  -o gpurun_out/prof_gate_$TAG python tools/profile_sweep.py > gpurun_out/ncu_gate_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_deep -c 1 \
  -o gpurun_out/prof_deep_$TAG python tools/layers_bench.py 5 > gpurun_out/ncu_deep_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sweep_general -c 1 \
  -o gpurun_out/prof_general_$TAG python tools/layers_bench.py 3 > gpurun_out/ncu_general_$TAG.log 2>&1
./tools/rfbench > gpurun_out/rfbench_$TAG.txt 2>&1
./tools/dmma_bench > gpurun_out/dmma_$TAG.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo done
# keep the copy-back under gpurun's 64 MiB: raw pages as CSV, the reports themselves dropped
for k in sweep gate deep general; do
  [ -f gpurun_out/prof_${k}_$TAG.ncu-rep ] && ncu -i gpurun_out/prof_${k}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_${TAG}_raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
