#!/bin/bash
# Build everything; non-zero exit (and the log tail) if the build fails -- so a GPU run never
# measures a stale library.
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /tmp/es_build.log 2>&1 || { tail -5 /tmp/es_build.log; exit 1; }
echo "build ok"
