#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune5; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
V="k=warp;k=warp,U=16;k=tma,st=4;k=tma,st=8;k=tma,st=3"
timeout 900 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
timeout 900 python scripts/tune.py --config proteins --F 128 --reduce sum --variants "$V" > $OUT/proteins128.jsonl 2>&1
timeout 900 python scripts/tune.py --config arxiv --F 128 --s 64 --reduce sum --variants "$V" > $OUT/arxiv128.jsonl 2>&1
timeout 900 python scripts/tune.py --config reddit --F 602 --variants "k=tma,st=4;k=tma,st=3;k=tma,st=4,m=24;k=tma,st=8" > $OUT/reddit602.jsonl 2>&1
