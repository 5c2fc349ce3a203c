#!/bin/bash
# One measurement pass on one GPU (round 2): smoke, optional GPU tests, a bench line per config
# (cold L2; Reddit also warm, Bucket and bf16), the reference arm, the ncu launch list of a Reddit
# step, and one ncu --set full capture of the dominant kernel's launches of ONE step per config
# (summaries feed profiles/ncu_traffic.json via scripts/traffic_table.py).
# Usage (from this container): gpurun --timeout 3600 -- 'bash scripts/gpu_pass.sh <tag>'
#   SKIP_TESTS=1 / SKIP_NCU=1 / SKIP_SAN=1
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02}; OUT=gpurun_out/$TAG; mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 3000 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
B="timeout 900 python bench.py"
$B > "$OUT/bench_reddit602.json" 2> "$OUT/bench.err"
$B --no-flush --no-e2e --no-cpu-baseline > "$OUT/bench_reddit602_warm.json" 2>> "$OUT/bench.err"
$B --strategy bucket --no-e2e --no-cpu-baseline > "$OUT/bench_reddit602_bucket.json" 2>> "$OUT/bench.err"
$B --bf16 --no-e2e --no-cpu-baseline > "$OUT/bench_reddit602_bf16.json" 2>> "$OUT/bench.err"
$B --config reddit --F 128 > "$OUT/bench_reddit128.json" 2>> "$OUT/bench.err"
for c in proteins arxiv pubmed scaled; do $B --config $c > "$OUT/bench_$c.json" 2>> "$OUT/bench.err"; done
timeout 600 python bench.py --impl reference --steps 3 > "$OUT/ref_reddit602.json" 2> "$OUT/ref.err"
timeout 1200 python scripts/s_sweep.py > "$OUT/s_sweep.jsonl" 2> "$OUT/s_sweep.err"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches_reddit602.csv" \
      python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > "$OUT/ncu_launches.log" 2>&1
  # name : bench args : kernel regex : launches of it per step
  for spec in "reddit602::spmm_slab_flow:6" "reddit128:--config reddit --F 128:spmm_slab_flow:1" \
              "proteins:--config proteins:spmm_slab_flow:1" "arxiv:--config arxiv:spmm:1" \
              "pubmed:--config pubmed:spmm:1" "scaled:--config scaled:spmm:1"; do
    IFS=: read -r name args kre per <<< "$spec"
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kre -s $((3 * per)) -c $per \
        -o "$OUT/prof_$name" python bench.py $args --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --graph off \
        > "$OUT/ncu_$name.log" 2>&1
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
