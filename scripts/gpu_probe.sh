#!/bin/bash
# Slab-kernel A/B probe on one GPU (scripts/slab_probe.py), optional ncu capture of one pass.
# Usage (from this container): gpurun --timeout 1500 -- 'bash scripts/gpu_probe.sh <tag> "<variants>" [cfg F s strategy]...'
#   variants: kernel:stages:width:cta_warps:variant, comma-separated (see slab_probe.py)
#   NCU=<variant> additionally captures one pass of that variant with ncu --set full (reddit 602 256)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=$1; VARIANTS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p "$OUT"
[ $# -eq 0 ] && set -- "reddit 602 256 fastrand"
for spec in "$@"; do
  name=$(echo $spec | tr ' ' '_')
  SLAB_VARIANTS="$VARIANTS" timeout 900 python scripts/slab_probe.py $spec > "$OUT/probe_$name.jsonl" 2>> "$OUT/probe.err"
done
if [ -n "${NCU:-}" ]; then
  SLAB_VARIANTS=$NCU REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_slab -s 12 -c 1 \
     -o "$OUT/prof_ncu" python scripts/slab_probe.py reddit 602 256 > "$OUT/ncu.log" 2>&1
fi
tail -3 "$OUT/probe.err"
