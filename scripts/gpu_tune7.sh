#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune7; mkdir -p $OUT
V="k=warp;k=warp,U=2,m=4;k=warp,U=2,m=5;k=warp,U=2,m=6;k=warp,U=4,m=5;k=warp,U=4,m=6;k=warp"
timeout 900 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
timeout 900 python scripts/tune.py --config proteins --F 128 --reduce sum --variants "$V" > $OUT/proteins128.jsonl 2>&1
timeout 900 python scripts/tune.py --config arxiv --F 128 --s 64 --reduce sum --variants "$V" > $OUT/arxiv128.jsonl 2>&1
