#!/bin/bash
# ncu evidence for one workload: launch list (cold, serialised) + full sets of the top kernels.
W=${1:-C4}
OUT=gpurun_out
mkdir -p $OUT
CCDK_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$W.csv python tools/run_step.py $W 1 > $OUT/launches_$W.log 2>&1
CCDK_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_generation -s 30 -c 1 -o $OUT/prof_gen_$W -f python tools/run_step.py $W 0 > $OUT/prof_gen_$W.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_rows -c 1 -o $OUT/prof_sweep_$W -f python tools/run_step.py $W 0 > $OUT/prof_sweep_$W.log 2>&1
ls -la $OUT
