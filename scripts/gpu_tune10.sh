#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune10; mkdir -p $OUT
V="k=warp"; for d in 2 3 4 8; do for m in 4 6; do V="$V;k=cpasync,st=$d,m=$m"; done; done
timeout 900 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
timeout 900 python scripts/tune.py --config proteins --F 128 --reduce sum --variants "$V" > $OUT/proteins128.jsonl 2>&1
timeout 900 python scripts/tune.py --config arxiv --F 128 --s 64 --reduce sum --variants "$V" > $OUT/arxiv128.jsonl 2>&1
V="k=tma"; for d in 2 4 8; do for m in 1 4; do V="$V;k=cpasync,st=$d,m=$m"; done; done
timeout 900 python scripts/tune.py --config reddit --F 256 --variants "$V" > $OUT/reddit256.jsonl 2>&1
timeout 900 python scripts/tune.py --config reddit --F 200 --variants "$V" > $OUT/reddit200.jsonl 2>&1
V="k=tma;k=cpasync,st=2;k=cpasync,st=4"
timeout 900 python scripts/tune.py --config reddit --F 384 --variants "$V" > $OUT/reddit384.jsonl 2>&1
timeout 900 python scripts/tune.py --config reddit --F 512 --variants "$V" > $OUT/reddit512.jsonl 2>&1
