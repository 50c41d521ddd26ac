#!/bin/bash
# On the GPU box: one ncu --set full capture of the f16 engine (tools/prec_probe.py,
# second float launch) into gpurun_out/prof_f16.ncu-rep.
ncu --set full --clock-control none --import-source on -k regex:k_decode_flt -s 1 -c 1 -o gpurun_out/prof_f16 python tools/prec_probe.py > gpurun_out/ncu_f16.log 2>&1; echo rc $?
