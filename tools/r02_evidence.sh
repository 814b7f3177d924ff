#!/bin/bash
# Round-2 evidence pass on one B200 (run under gpurun): multi-GPU device test,
# per-rank scaling prediction, launch list with DRAM bytes, sanitizers.
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_multigpu_device.py -m gpu -q > $OUT/mgpu_device.log 2>&1; echo "mgpu rc=$?"
timeout 600 python tools/predict_scaling.py --out $OUT/predict_C4.json > $OUT/predict_C4.log 2>&1; echo "predict rc=$?"
CCDK_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/launches_dram_C4.csv python tools/run_step.py C4 1 > $OUT/launches_dram_C4.log 2>&1; echo "ncu rc=$?"
for tool in racecheck synccheck memcheck; do
  CCDK_NO_GRAPH=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/san_step.py > $OUT/san_$tool.log 2>&1; echo "san $tool rc=$?"
done
(cd $OUT && CCDK_NO_GRAPH=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 ../tests/cpp/_reftests/test_pipeline > san_memcheck_dropin.log 2>&1; echo "san dropin rc=$?")
