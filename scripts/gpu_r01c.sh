#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/r01c; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --config scaled > $OUT/bench_scaled.json 2> $OUT/bench_scaled.err
for c in arxiv proteins pubmed; do timeout 600 python bench.py --config $c --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
timeout 600 python bench.py --config reddit --F 128 --no-e2e > $OUT/bench_reddit128.json 2> $OUT/bench_reddit128.err
ES_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench_gloo2.json 2> $OUT/bench_gloo2.err
ES_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > $OUT/ref_gloo2.json 2> $OUT/ref_gloo2.err
