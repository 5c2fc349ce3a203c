#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/tune11; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "rowgroup" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
V="k=subwarp;k=rowgroup;k=rowgroup,U=8;k=subwarp"
timeout 600 python scripts/tune.py --config pubmed --F 16 --s 32 --reduce sum --strategy bucket --variants "$V" > $OUT/pubmed.jsonl 2>&1
timeout 600 python scripts/tune.py --config arxiv --F 16 --s 64 --reduce sum --variants "$V" > $OUT/arxiv16.jsonl 2>&1
timeout 600 python scripts/tune.py --config reddit --F 16 --variants "$V" > $OUT/reddit16.jsonl 2>&1
