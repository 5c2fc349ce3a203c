#!/bin/bash
# Kernel-variant sweep on one GPU: prints config + ms_per_step + roofline frac per line.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out/${1:-sweep}; shift || true
mkdir -p "$OUT"
run() {  # run <label> <env...> -- <bench args>
  local label=$1; shift
  local envs=(); while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  env "${envs[@]}" timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 "$@" > "$OUT/$label.json" 2> "$OUT/$label.err"
  python - "$OUT/$label.json" "$label" <<'PY'
import json,sys
try:
    j=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:40s} {j['ms_per_step']:9.3f} ms  {j['value']:9.1f} GF/s  frac {j['roofline']['frac']:.3f}  {j['roofline']['kernel']}")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
}
source "${SWEEP_SPEC:-scripts/sweep_spec.sh}"
