#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune3; mkdir -p $OUT
V="k=tma,st=4,m=1"
for h in 400 600 800 1000 1300; do V="$V;k=tma,st=4,m=1,hot=$h;k=tma,st=4,m=16,hot=$h;k=tma,st=3,m=1,hot=$h"; done
V="$V;k=tma,st=4,m=1"
timeout 900 python scripts/tune.py --config reddit --F 602 --steps 8 --variants "$V" > $OUT/reddit602_hot.jsonl 2>&1
V="k=tma,st=4,m=1"; for h in 300 500 800 1200; do V="$V;k=tma,st=4,m=1,hot=$h"; done
timeout 600 python scripts/tune.py --config reddit --F 256 --steps 8 --variants "$V" > $OUT/reddit256_hot.jsonl 2>&1
