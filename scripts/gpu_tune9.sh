#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune9; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "cpasync" > $OUT/pytest_cpasync.log 2>&1; echo "rc=$?" >> $OUT/pytest_cpasync.log
V="k=warp"; for d in 2 3 4 8; do for m in 6 8; do V="$V;k=cpasync,st=$d,m=$m"; done; done
timeout 900 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
timeout 900 python scripts/tune.py --config proteins --F 128 --reduce sum --variants "$V" > $OUT/proteins128.jsonl 2>&1
timeout 900 python scripts/tune.py --config arxiv --F 128 --s 64 --reduce sum --variants "$V" > $OUT/arxiv128.jsonl 2>&1
V="k=tma;k=cpasync,st=2;k=cpasync,st=4;k=tma"
timeout 900 python scripts/tune.py --config reddit --F 256 --variants "$V" > $OUT/reddit256.jsonl 2>&1
timeout 900 python scripts/tune.py --config reddit --F 602 --variants "$V" > $OUT/reddit602.jsonl 2>&1
