#!/bin/bash
# round-2 first GPU pass: new dispatch tests, the parity suite, smoke, a short bench
T=${1:-r2a}
timeout 1500 python -m pytest tests/test_gpu_dispatch.py -q > gpurun_out/${T}_dispatch.log 2>&1; echo "dispatch rc=$?"; tail -15 gpurun_out/${T}_dispatch.log
timeout 1200 python -m pytest tests -m gpu -q --deselect tests/test_gpu_dispatch.py > gpurun_out/${T}_parity.log 2>&1; echo "parity rc=$?"; tail -8 gpurun_out/${T}_parity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${T}_smoke.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("gpurun_out/${T}_bench.log").read().strip().splitlines()[-1])
print("value %.4g" % d["value"], {m: ("%.3g/s" % v["normals_per_s"], "%.3f ms" % v["ms_per_call"]) for m, v in d["per_method"].items()}, d["clocks"])
PY
