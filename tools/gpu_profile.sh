#!/bin/bash
# Run on the GPU box (via gpurun): plain bench, launch list, full capture of
# the sweep kernel.  Outputs land in gpurun_out/ (summarised by
# tools/ncu_summary.py into profiles/).
set -u
TAG=${1:-r01}
EXTRA=${2:-}
CMD="python bench.py --steps 6 --warmup 3 --no-cpu --no-secondary $EXTRA"
mkdir -p gpurun_out
python bench.py $EXTRA > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -1 gpurun_out/bench_${TAG}.json
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD \
    > gpurun_out/ncu_launch_${TAG}.log 2>&1
$CMD > gpurun_out/plain2_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 \
    -o gpurun_out/sweep_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
