#!/usr/bin/env bash
# Build the current tree's library as paper_2406_14424_b200/lib_ab_$1.so (for
# same-box A/B timing through GS_LIB_PATH), then restore the normal build.
set -e
python -c "from paper_2406_14424_b200 import _build; _build.build()" > /dev/null
cp paper_2406_14424_b200/libgearserve_b200.so "paper_2406_14424_b200/lib_ab_$1.so"
