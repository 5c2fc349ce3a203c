#!/bin/bash
# One GPU round: L2 peak probe, smoke, gpu tests, bench, ncu launch list + full capture of the hot kernel.
# Usage (from this container): gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh <tag> [bench args...]'
#   SKIP_TESTS=1 / SKIP_NCU=1 / L2PEAK=1 (re-measure profiles/l2_peak.json into gpurun_out/<tag>/)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r02}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
if [ "${L2PEAK:-0}" = "1" ]; then
  timeout 300 python scripts/l2_peak.py "$OUT/l2_peak.json" > "$OUT/l2_peak.log" 2>&1
  cp "$OUT/l2_peak.json" profiles/l2_peak.json 2>/dev/null
fi
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
fi
timeout 900 python bench.py "$@" > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
      python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > "$OUT/ncu_launches.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -s 3 -c 1 \
      -o "$OUT/prof" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > "$OUT/ncu_full.log" 2>&1
  python scripts/ncu_summary.py "$OUT/prof.ncu-rep" > "$OUT/prof.summary.jsonl" 2>&1
fi
du -sh "$OUT"
