#!/bin/bash
# One gpurun call re-establishing the round-2 evidence: GPU tests + smoke, the bench line and
# the reference arm, the bench's ncu launch list, full ncu captures of the config-4 sweep and
# the gate build, the small-job probe (BASELINE C1 / C2 / C5), per-config e2e, L = 1..8
# throughput and the pair-list kernel.
# usage: gpurun --timeout 3000 -- 'bash tools/gpu_round_r2.sh r2e'
TAG=${1:-r2e}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nproc > gpurun_out/host_$TAG.txt; lscpu >> gpurun_out/host_$TAG.txt; nvidia-smi >> gpurun_out/host_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 300 python tools/gate_bench.py > gpurun_out/gate_bench_$TAG.jsonl 2>&1
timeout 600 python tools/small_jobs.py > gpurun_out/small_jobs_$TAG.jsonl 2> gpurun_out/small_jobs_$TAG.err
timeout 600 python tools/configs_e2e.py > gpurun_out/configs_e2e_$TAG.jsonl 2>&1
timeout 600 python tools/layers_bench.py 1 2 3 4 5 6 7 8 5:784:512 6:784:192 7:128:256 > gpurun_out/layers_$TAG.jsonl 2>&1
timeout 300 python tools/pairs_bench.py > gpurun_out/pairs_$TAG.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 \
  -o gpurun_out/prof_sweep_$TAG python tools/profile_sweep.py > gpurun_out/ncu_sweep_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gate_build -c 1 \
  -o gpurun_out/prof_gate_$TAG python tools/gate_bench.py > gpurun_out/ncu_gate_$TAG.log 2>&1
for k in sweep gate; do
  [ -f gpurun_out/prof_${k}_$TAG.ncu-rep ] && ncu -i gpurun_out/prof_${k}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_${TAG}_raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep
echo done
