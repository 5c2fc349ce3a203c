#!/bin/bash
# compute-sanitizer over every kernel family incl. the slab path; 2-rank bench flow (gloo, ranks
# sharing cuda:0 -- validation only) on the slab path.
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/r01m; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $tool python scripts/sanitize.py (slab path included)" >> $OUT/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py >> $OUT/sanitizer.txt 2>&1; echo "rc=$?" >> $OUT/sanitizer.txt
done
ES_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > $OUT/bench_gloo2.json 2> $OUT/bench_gloo2.err
echo "torchrun rc=$?" >> $OUT/bench_gloo2.err
