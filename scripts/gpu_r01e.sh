#!/bin/bash
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/r01e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench_reddit602.json 2> $OUT/bench_reddit602.err
for c in arxiv proteins pubmed; do timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
timeout 600 python bench.py --config reddit --F 128 > $OUT/bench_reddit128.json 2> $OUT/bench_reddit128.err
timeout 900 python bench.py --config scaled > $OUT/bench_scaled.json 2> $OUT/bench_scaled.err
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize.py > $OUT/sanitize_memcheck.log 2>&1; echo "rc=$?" >> $OUT/sanitize_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize.py > $OUT/sanitize_racecheck.log 2>&1; echo "rc=$?" >> $OUT/sanitize_racecheck.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 3 -c 1 -o $OUT/prof128 python bench.py --config reddit --F 128 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu128.log 2>&1
python scripts/ncu_summary.py $OUT/prof128.ncu-rep > $OUT/prof128.summary.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 3 -c 1 -o $OUT/prof256 python bench.py --config scaled --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu256.log 2>&1
python scripts/ncu_summary.py $OUT/prof256.ncu-rep > $OUT/prof256.summary.jsonl 2>&1
rm -f $OUT/prof256.ncu-rep
du -sh $OUT
