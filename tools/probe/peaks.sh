#!/bin/bash
# Measure the FP64 and HBM-write peaks (burst + sustained) with clocks sampled alongside.
# usage (on the GPU box): bash tools/probe/peaks.sh TAG  -> gpurun_out/TAG_peaks.json, TAG_peaks_clocks.csv
TAG=${1:-peaks}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/probe/peaks.cu || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap \
    --format=csv,noheader,nounits -lms 100 > gpurun_out/${TAG}_peaks_clocks.csv &
SMI=$!
/tmp/peaks > gpurun_out/${TAG}_peaks.json
RC=$?
kill $SMI; wait $SMI 2>/dev/null
cat gpurun_out/${TAG}_peaks.json
exit $RC
