#!/bin/bash
# e2e phase traces of the joint host pipeline for libqk variants (VARIANTS="0 1 2", 0 = libqk.so).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
OUT=gpurun_out/${1:-e2evar}.txt
for V in ${VARIANTS:-0 1 2}; do
  LIBV=$PWD/paper_2405_02630_b200/_lib/libqk_v$V.so; [ "$V" = 0 ] && LIBV=$PWD/paper_2405_02630_b200/_lib/libqk.so
  echo "== v$V" >> $OUT
  QK_LIB_PATH=$LIBV timeout 300 python tools/e2e_joint_probe.py 4 >> $OUT 2>&1
  QK_LIB_PATH=$LIBV timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench v$V', round(d['value']/1e9,4), round(d['e2e']['value']/1e9,4), d['clocks']['sm_mhz'])" >> $OUT
done
echo done >> $OUT
