#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/prof3; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'spmm_warp|csrmm|SpMM|spmm' -s 4 -c 2 -o $OUT/f128 python scripts/prof_f128.py reddit 256 > $OUT/f128.log 2>&1
python scripts/ncu_summary.py $OUT/f128.ncu-rep > $OUT/f128.summary.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'spmm_warp|csrmm|SpMM|spmm' -s 4 -c 2 -o $OUT/arxiv python scripts/prof_f128.py arxiv 64 > $OUT/arxiv.log 2>&1
python scripts/ncu_summary.py $OUT/arxiv.ncu-rep > $OUT/arxiv.summary.jsonl 2>&1
rm -f $OUT/arxiv.ncu-rep
