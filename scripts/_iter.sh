set -u
cd "${GRAFT_REPO_ROOT}"
OUT=gpurun_out/r02s12; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo "build rc=$?" >> $OUT/build.log
timeout 900 python -m pytest tests/test_gpu_slab.py -x -q > $OUT/pytest_slab.log 2>&1; echo "rc=$?" >> $OUT/pytest_slab.log
V="slab_smem,slab_flow,slab_flow:0:0:8,slab_flow:0:16:8"
SLAB_VARIANTS=$V timeout 600 python scripts/slab_probe.py reddit 602 256 fastrand > $OUT/probe_reddit602.jsonl 2> $OUT/probe.err
SLAB_VARIANTS=$V timeout 600 python scripts/slab_probe.py reddit 602 256 bucket > $OUT/probe_reddit602_bucket.jsonl 2>> $OUT/probe.err
SLAB_VARIANTS=$V timeout 600 python scripts/slab_probe.py reddit 128 256 fastrand > $OUT/probe_reddit128.jsonl 2>> $OUT/probe.err
SLAB_VARIANTS=$V timeout 600 python scripts/slab_probe.py proteins 128 256 fastrand > $OUT/probe_proteins.jsonl 2>> $OUT/probe.err
SLAB_VARIANTS=$V timeout 600 python scripts/slab_probe.py reddit 602 64 fastrand > $OUT/probe_reddit602_s64.jsonl 2>> $OUT/probe.err
SLAB_VARIANTS=$V timeout 600 python scripts/slab_probe.py arxiv 128 64 fastrand > $OUT/probe_arxiv.jsonl 2>> $OUT/probe.err
timeout 600 python bench.py > $OUT/bench_reddit602.json 2> $OUT/bench.err
tail -2 $OUT/pytest_slab.log
