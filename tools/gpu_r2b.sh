#!/bin/bash
# round 2, second GPU pass: peaks probe, full bench line, racecheck over every kernel path
T=${1:-r2b}
bash tools/probe/peaks.sh $T > /dev/null 2>&1; echo "peaks rc=$?"; cat gpurun_out/${T}_peaks.json
cp gpurun_out/${T}_peaks.json profiles/peaks.json 2>/dev/null
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/${T}_bench.log | tail -3 | cut -c1-1500
timeout 300 python tools/dispatch_cases.py > gpurun_out/${T}_plain.log 2>&1 && \
  timeout 1800 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 200 python tools/dispatch_cases.py > gpurun_out/${T}_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/${T}_racecheck.log
