#!/bin/bash
# ncu capture of the configs' own launches (C1 B1, C2 P, C3 B3, C4 2^22) with the current build
T=${1:-r2m}
python tools/profile_configs.py > gpurun_out/${T}_cfg_plain.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:"pw_kernel|b3_kernel|mid_kernel" -o gpurun_out/${T}_cfg python tools/profile_configs.py > gpurun_out/${T}_cfg_ncu.log 2>&1; echo "cfg ncu rc=$?"
