#!/bin/bash
# Full bench line + reference arm + the ncu launch list of the same bench command.
TAG=${1:-full}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_full_$TAG.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --validate 0 --configs 0 > gpurun_out/bench_short_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --validate 0 --configs 0 > gpurun_out/ncu_launches_$TAG.log 2>&1; echo "ncu rc=$?"
tail -c 3000 gpurun_out/bench_full_$TAG.log
