#!/bin/bash
# One GPU iteration: parity tests, a short bench, and an ncu capture of the four hot kernels.
# usage: bash tools/gpu_iter.sh TAG [pytest-args]
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/bench_$TAG.log").read().strip().splitlines()[-1])
print("value %.4g" % d["value"], {m: ("%.3g/s" % v["normals_per_s"], "%.3f ms" % v["ms_per_call"]) for m, v in d["per_method"].items()}, d["clocks"])
PY
if [ "${NCU:-1}" = "1" ]; then
python tools/profile_step.py > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"pw_kernel|b3_kernel|polar" -s 7 -c 7 -o gpurun_out/prof_$TAG python tools/profile_step.py > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
fi
