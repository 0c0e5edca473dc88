#!/bin/bash
# Kernel-variant sweep: libqk_v*.so builds x QK_SWEEP_RI, bench value + FP64 pipe fraction.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
OUT=gpurun_out/${1:-var}.txt
for rep in 1 2; do for V in ${VARIANTS:-1 2 3 4 5 6}; do for RI in ${RIS:-4 2}; do
QK_SWEEP_RI=$RI QK_LIB_PATH=$PWD/paper_2405_02630_b200/_lib/libqk_v$V.so timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('v$V', $RI, round(d['value']/1e9,4), round(d['roofline']['fp64_pipe_frac'],4), d['clocks']['sm_mhz'])" >> $OUT
done; done; done
