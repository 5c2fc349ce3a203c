#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune1; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
V="warp"; for st in 4 8 16; do for r in 1 2 4 8 16 32; do V="$V;tma:$st:$r"; done; done
timeout 600 python scripts/tune.py --config reddit --F 602 --variants "$V" > $OUT/reddit602.jsonl 2>&1
V="warp"; for st in 8 16; do for r in 2 4 8 16 32; do V="$V;tma:$st:$r"; done; done
timeout 600 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
timeout 600 python scripts/tune.py --config proteins --F 128 --reduce sum --variants "$V" > $OUT/proteins128.jsonl 2>&1
timeout 600 python scripts/tune.py --config arxiv --F 128 --s 64 --reduce sum --variants "$V" > $OUT/arxiv128.jsonl 2>&1
