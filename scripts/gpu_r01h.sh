#!/bin/bash
# Re-entry check: smoke, GPU tests, default bench, L2/DRAM bandwidth probe.
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/r01h; mkdir -p $OUT
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/l2bw scripts/l2bw.cu && timeout 300 /tmp/l2bw > $OUT/l2bw.jsonl 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_reddit602.json 2> $OUT/bench_reddit602.err
