#!/bin/bash
# Full measurement pass on one GPU: smoke, all GPU tests, bench lines for every config (cold and
# warm L2), the reference arm, ncu launch list + full capture per config, compute-sanitizer.
# Usage (from this container): gpurun --timeout 5400 -- 'bash scripts/gpu_measure.sh <tag>'
#   SKIP_TESTS=1 / SKIP_NCU=1 / SKIP_SAN=1
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 3000 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
timeout 900 python bench.py > "$OUT/bench_reddit602.json" 2> "$OUT/bench_reddit602.err"
timeout 600 python bench.py --no-flush --no-e2e --no-cpu-baseline > "$OUT/bench_reddit602_warm.json" 2>> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 3 > "$OUT/ref_reddit602.json" 2> "$OUT/ref_reddit602.err"
for c in arxiv proteins pubmed; do timeout 600 python bench.py --config $c > "$OUT/bench_$c.json" 2>> "$OUT/bench.err"; done
timeout 600 python bench.py --config reddit --F 128 > "$OUT/bench_reddit128.json" 2>> "$OUT/bench.err"
timeout 900 python bench.py --config scaled > "$OUT/bench_scaled.json" 2>> "$OUT/bench.err"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_reddit602.csv" \
      python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
  for spec in "reddit602:--config reddit" "reddit128:--config reddit --F 128" "proteins:--config proteins" "arxiv:--config arxiv" "pubmed:--config pubmed" "scaled:--config scaled"; do
    name=${spec%%:*}; args=${spec#*:}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 3 -c 1 -o "$OUT/prof_$name" \
        python bench.py $args --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --graph off > "$OUT/ncu_$name.log" 2>&1
    python scripts/ncu_summary.py "$OUT/prof_$name.ncu-rep" > "$OUT/prof_$name.summary.jsonl" 2>&1
    [ "$name" != "reddit602" ] && rm -f "$OUT/prof_$name.ncu-rep"
  done
fi
if [ "${SKIP_SAN:-0}" != "1" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize.py > "$OUT/sanitize_$tool.log" 2>&1
    echo "rc=$?" >> "$OUT/sanitize_$tool.log"
  done
fi
du -sh "$OUT"
