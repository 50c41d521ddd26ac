#!/bin/bash
# Run on the GPU box (via gpurun): plain bench run, launch list, one full ncu
# capture of the decode kernel. Outputs land in gpurun_out/.
set -u
TAG=${1:-r01}
ARGS="--steps 2 --warmup 1 --no-e2e --no-cpu"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 1 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
