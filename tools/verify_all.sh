#!/bin/bash
# One-shot verification on a B200 box (what the round-end driver runs):
#   build -> CPU tests -> GPU tests -> smoke -> bench (C4) -> reference arm.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- bash tools/verify_all.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/verify_build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m "not gpu" -q 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py 2> gpurun_out/verify_bench.err | tail -1 | tee gpurun_out/verify_bench.json | cut -c1-160
timeout 600 python bench.py --impl reference 2>&1 | tail -1 | cut -c1-160
