#!/bin/bash
T=r2q
python tools/profile_step.py --methods B1 > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pw_kernel" -s 1 -c 1 -o gpurun_out/${T}_b1 python tools/profile_step.py --methods B1 > gpurun_out/${T}_ncu1.log 2>&1; echo rc=$?
NRNG_LIB_OVERRIDE=ab_libs/b1unroll.so python tools/profile_step.py --methods B1 > gpurun_out/${T}_plain2.log 2>&1 && \
NRNG_LIB_OVERRIDE=ab_libs/b1unroll.so ncu --set full --clock-control none --import-source on -k regex:"pw_kernel" -s 1 -c 1 -o gpurun_out/${T}_b1u python tools/profile_step.py --methods B1 > gpurun_out/${T}_ncu2.log 2>&1; echo rc=$?
