#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune12; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "halfwarp" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
V="k=cpasync;k=cpasync,HALFWARP=1;k=cpasync,HALFWARP=1,m=5;k=cpasync,HALFWARP=1,st=8;k=cpasync,HALFWARP=1,st=2,m=5;k=cpasync"
timeout 600 python scripts/tune.py --config reddit --F 128 --variants "$V" > $OUT/reddit128.jsonl 2>&1
timeout 600 python scripts/tune.py --config proteins --F 128 --reduce sum --variants "$V" > $OUT/proteins128.jsonl 2>&1
timeout 600 python scripts/tune.py --config arxiv --F 128 --s 64 --reduce sum --variants "$V" > $OUT/arxiv128.jsonl 2>&1
timeout 600 python scripts/tune.py --config reddit --F 64 --variants "$V" > $OUT/reddit64.jsonl 2>&1
