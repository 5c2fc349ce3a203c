#!/bin/bash
# slab path: GPU tests + bench (auto = slab for Reddit F=602) + fused A/B
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/r01i; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_reddit602.json 2> $OUT/bench_reddit602.err
timeout 600 python bench.py --kernel fused --no-e2e --no-cpu-baseline > $OUT/bench_reddit602_fused.json 2> $OUT/bench_reddit602_fused.err
timeout 600 python bench.py --F 128 --kernel slab --no-e2e --no-cpu-baseline > $OUT/bench_reddit128_slab.json 2> $OUT/bench_reddit128_slab.err
