#!/bin/bash
# Per-generation cost of the narrow phase: intervals per generation (CCDK_GEN_TRACE)
# and each k_generation / k_finish launch's duration (ncu, direct launches).
W=${1:-C4}
OUT=gpurun_out
mkdir -p $OUT
CCDK_GEN_TRACE=1 python tools/run_step.py $W 0 > $OUT/gens_$W.log 2>&1
CCDK_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'k_generation|k_finish|k_gen0|k_classify_gen0' \
  --log-file $OUT/genlaunch_$W.csv python tools/run_step.py $W 0 > $OUT/genlaunch_$W.log 2>&1
