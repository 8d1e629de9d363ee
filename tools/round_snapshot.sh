#!/bin/bash
# Everything the round's record needs, in one GPU session: tests, full bench line (+e2e,
# cpu baseline), the reference arm, per-config numbers, launch list, ncu --set full capture.
TAG=${1:-snap}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
bash tools/bench_full.sh $TAG > /dev/null 2>&1; echo "bench_full done"
timeout 900 python tools/bench_configs.py > gpurun_out/configs_$TAG.json 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"
python tools/profile_step.py > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"pw_kernel|b3_kernel|polar" -s 7 -c 7 -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
# the launch list of every dispatch path (each kernel instantiation nrng.cu launches)
python tools/dispatch_cases.py > gpurun_out/disp_plain_$TAG.log 2>&1 && \
 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dispatch_launches_$TAG.csv python tools/dispatch_cases.py > gpurun_out/disp_ncu_$TAG.log 2>&1; echo "dispatch ncu rc=$?"
