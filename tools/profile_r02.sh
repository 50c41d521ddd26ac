#!/bin/bash
# Round-2 profiling on the GPU box (via gpurun); outputs in gpurun_out/.
#  1. headline: plain bench run, ncu launch list, one --set full capture of the decode kernel
#  2. f16 engine on the headline shape (--set full)
#  3. config 4 mixed batch: every per-shape kernel of one replay (SpeedOfLight/Occupancy/Launch)
set -u
TAG=${1:-r02}
ARGS="--steps 3 --warmup 3 --no-e2e --no-cpu --no-configs"
mkdir -p gpurun_out
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_decode_i8 -s 3 -c 1 \
    -o gpurun_out/prof_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_decode_flt -s 1 -c 1 \
    -o gpurun_out/prof_f16_$TAG python tools/prec_probe.py > gpurun_out/ncu_f16_$TAG.log 2>&1
echo "f16 rc=$?"
python tools/prof_config4.py 30 > gpurun_out/cfg4_plain_$TAG.log 2>&1
ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section SchedulerStats \
    --clock-control none -k regex:k_decode -s 204 -c 102 \
    -o gpurun_out/prof_cfg4_$TAG python tools/prof_config4.py 1 > gpurun_out/ncu_cfg4_$TAG.log 2>&1
echo "cfg4 rc=$?"
