#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune4; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
V="k=warp"
for r in 4 8 16 32; do for u in 4 8 16; do for m in 1 2 3; do V="$V;k=stream,r=$r,U=$u,m=$m"; done; done; done
timeout 900 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
timeout 900 python scripts/tune.py --config proteins --F 128 --reduce sum --variants "$V" > $OUT/proteins128.jsonl 2>&1
timeout 900 python scripts/tune.py --config arxiv --F 128 --s 64 --reduce sum --variants "$V" > $OUT/arxiv128.jsonl 2>&1
