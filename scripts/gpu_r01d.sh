#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/r01d; mkdir -p $OUT
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > $OUT/sanitize_$tool.log 2>&1; echo "rc=$?" >> $OUT/sanitize_$tool.log
done
timeout 900 python scripts/vs_cusparse.py reddit 602 > $OUT/vs_cusparse_reddit602.jsonl 2>&1
timeout 900 python scripts/vs_cusparse.py reddit 128 > $OUT/vs_cusparse_reddit128.jsonl 2>&1
timeout 900 python scripts/vs_cusparse.py proteins 128 > $OUT/vs_cusparse_proteins128.jsonl 2>&1
