#!/usr/bin/env bash
# Build phase-timing variants of the library here (nvcc cross-compiles), run
# tools/phase_probe.py against each on the GPU box: VARIANTS="tag:DEFINE ..."
set -e
cd "$(dirname "$0")/.."
for v in $VARIANTS; do
  tag=${v%%:*}; def=${v#*:}
  python - <<PY
from paper_2406_14424_b200 import _build
d = tuple(x for x in "$def".split(",") if x)
print(_build.build(phase_timing=True, defines=d, tag="_$tag"))
PY
done
