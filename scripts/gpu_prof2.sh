#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/prof2; mkdir -p $OUT
i=0
for V in "k=tma,st=4,m=1" "k=tma,st=4,m=24" "k=tma,st=4,m=24,hot=800" "k=tma,st=8,m=1"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm -s 2 -c 1 -o $OUT/v$i \
    python scripts/tune.py --config reddit --F 602 --steps 1 --variants "$V" > $OUT/v$i.log 2>&1
done
for i in 1 2 3 4; do python scripts/ncu_summary.py $OUT/v$i.ncu-rep > $OUT/v$i.summary.jsonl 2>&1; done
for i in 2 3 4; do rm -f $OUT/v$i.ncu-rep; done
du -sh gpurun_out
