#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune2; mkdir -p $OUT
V="k=warp"
for st in 2 3 4 6 8; do for m in 1 16 24 32; do V="$V;k=tma,st=$st,m=$m"; done; done
for r in 2 4; do V="$V;k=tma,st=4,m=24,r=$r;k=tma,st=3,m=32,r=$r"; done
timeout 900 python scripts/tune.py --config reddit --F 602 --variants "$V" > $OUT/reddit602.jsonl 2>&1
V="k=tma,st=4,m=24"; for h in 100 200 300 500 800 1200 2000; do V="$V;k=tma,st=4,m=24,hot=$h"; done
timeout 600 python scripts/tune.py --config reddit --F 602 --variants "$V" > $OUT/reddit602_hot.jsonl 2>&1
V="k=warp"; for st in 3 4 6 8; do for m in 16 24 32; do V="$V;k=tma,st=$st,m=$m"; done; done
timeout 600 python scripts/tune.py --config reddit --F 256 --variants "$V" > $OUT/reddit256.jsonl 2>&1
V="k=warp"; for st in 4 8; do for m in 24 32; do V="$V;k=tma,st=$st,m=$m,TMA_MIN_BYTES=0"; done; done
timeout 600 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
