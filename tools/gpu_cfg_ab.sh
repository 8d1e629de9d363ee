#!/bin/bash
# interleaved per-config A/B: bash tools/gpu_cfg_ab.sh ROUNDS LIB...
R=$1; shift
for r in $(seq $R); do for lib in "$@"; do
  if [ $lib = default ]; then unset NRNG_LIB_OVERRIDE; else export NRNG_LIB_OVERRIDE=$lib; fi
  python tools/cfg_ab.py
done; done
