#!/bin/bash
# Measurement pass after the slab path: smoke, GPU tests, bench for every config, ncu launch
# list of the default bench command, ncu --set full of one whole step for the slab configs.
cd "${GRAFT_REPO_ROOT}"
TAG=${1:-r01j}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_reddit602.json 2> $OUT/bench_reddit602.err
timeout 600 python bench.py --impl reference --steps 3 > $OUT/ref_reddit602.json 2> $OUT/ref_reddit602.err
for c in arxiv proteins pubmed; do timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
timeout 600 python bench.py --config reddit --F 128 > $OUT/bench_reddit128.json 2> $OUT/bench_reddit128.err
timeout 900 python bench.py --config scaled > $OUT/bench_scaled.json 2> $OUT/bench_scaled.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_reddit602.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launches.log 2>&1
for spec in "reddit602:56:14:--config reddit" "reddit128:24:6:--config reddit --F 128" "proteins:24:6:--config proteins"; do
  IFS=: read name skip cnt args <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"slab|sample|Scan" -s $skip -c $cnt \
      -o $OUT/step_$name python bench.py $args --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --graph off > $OUT/ncu_$name.log 2>&1
  python scripts/ncu_step.py $OUT/step_$name.ncu-rep > $OUT/step_$name.json 2>&1
  python scripts/ncu_summary.py $OUT/step_$name.ncu-rep > $OUT/step_$name.summary.jsonl 2>&1
  [ "$name" != "reddit602" ] && rm -f $OUT/step_$name.ncu-rep
done
du -sh $OUT
timeout 1200 python scripts/s_sweep.py > $OUT/s_sweep.jsonl 2> $OUT/s_sweep.err
timeout 600 python scripts/e2e_gnn.py > $OUT/e2e_gnn.jsonl 2> $OUT/e2e_gnn.err
