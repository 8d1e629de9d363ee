#!/bin/bash
# GPU call: parity of the in-tree build (dispatch + parity suites), then an interleaved A/B
# of library variants at the bench shape.  usage: bash tools/gpu_ab.sh TAG ROUNDS METHODS LIB...
T=$1; R=$2; M=$3; shift 3
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
fi
AB_WARM=${AB_WARM:-25} bash tools/ab_rounds.sh $R $M "$@" 2>&1 | tee gpurun_out/${T}_ab.log
