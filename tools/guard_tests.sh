#!/bin/bash
# The GPU test suite with guard bands around every library buffer
# (MPB_GUARD=1, mpb_api.cu dev_alloc/dev_free): an out-of-bounds write by any
# kernel aborts the test process; an out-of-bounds read returns band bytes and
# breaks the bit-exact parity tests.  (compute-sanitizer is not available on
# the GPU pool.)
#   /usr/local/graft/bin/gpurun --timeout 1800 -- bash tools/guard_tests.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
MPB_GUARD=1 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider \
    > gpurun_out/guard_tests.log 2>&1
echo "guarded gpu tests rc=$? $(tail -1 gpurun_out/guard_tests.log)"
grep -m5 "MPB_GUARD: .*overwritten" gpurun_out/guard_tests.log || true
# the bands are really there: the library announces guard mode once
MPB_GUARD=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -m1 "MPB_GUARD"
