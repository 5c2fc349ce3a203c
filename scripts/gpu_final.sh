#!/bin/bash
# Full measurement pass: smoke, all GPU tests, bench lines for every config, ncu per config.
cd "${GRAFT_REPO_ROOT}"
TAG=${1:-r01g}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_reddit602.json 2> $OUT/bench_reddit602.err
timeout 600 python bench.py --impl reference --steps 3 > $OUT/ref_reddit602.json 2> $OUT/ref_reddit602.err
for c in arxiv proteins pubmed; do timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
timeout 600 python bench.py --config reddit --F 128 > $OUT/bench_reddit128.json 2> $OUT/bench_reddit128.err
timeout 900 python bench.py --config scaled > $OUT/bench_scaled.json 2> $OUT/bench_scaled.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_reddit602.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
for spec in "reddit602:--config reddit" "reddit128:--config reddit --F 128" "proteins:--config proteins" "arxiv:--config arxiv" "pubmed:--config pubmed" "scaled:--config scaled"; do
  name=${spec%%:*}; args=${spec#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 3 -c 1 -o $OUT/prof_$name \
      python bench.py $args --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --graph off > $OUT/ncu_$name.log 2>&1
  python scripts/ncu_summary.py $OUT/prof_$name.ncu-rep > $OUT/prof_$name.summary.jsonl 2>&1
  [ "$name" != "reddit602" ] && rm -f $OUT/prof_$name.ncu-rep
done
du -sh $OUT
