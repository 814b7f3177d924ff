#!/bin/bash
W=${1:-C4}; TAG=${2:-v2}
OUT=gpurun_out; mkdir -p $OUT
CCDK_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_generation -s 30 -c 1 -o $OUT/prof_gen_${W}_$TAG -f python tools/run_step.py $W 0 > $OUT/prof_gen_${W}_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep_rows -c 1 -o $OUT/prof_sweep_${W}_$TAG -f python tools/run_step.py $W 0 > $OUT/prof_sweep_${W}_$TAG.log 2>&1
ls $OUT
