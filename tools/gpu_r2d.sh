#!/bin/bash
# ncu captures: the configs' own launches (C1, C2, C3, C4 n=2^22), the bench-shape kernels, and the
# launch list of every dispatch path (tools/dispatch_cases.py)
T=${1:-r2d}
python tools/profile_configs.py > gpurun_out/${T}_cfg_plain.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:"pw_kernel|b3_kernel|mid_kernel|polar_kernel" -o gpurun_out/${T}_cfg python tools/profile_configs.py > gpurun_out/${T}_cfg_ncu.log 2>&1; echo "cfg ncu rc=$?"
python tools/dispatch_cases.py > gpurun_out/${T}_disp_plain.log 2>&1 && \
 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_dispatch_launches.csv python tools/dispatch_cases.py > gpurun_out/${T}_disp_ncu.log 2>&1; echo "dispatch ncu rc=$?"
python tools/profile_step.py --methods B1,B2,B3,P > gpurun_out/${T}_step_plain.log 2>&1 && \
 ncu --set full --clock-control none --import-source on -k regex:"pw_kernel|b3_kernel" -s 4 -c 4 -o gpurun_out/${T}_step python tools/profile_step.py --methods B1,B2,B3,P > gpurun_out/${T}_step_ncu.log 2>&1; echo "step ncu rc=$?"
ls -la gpurun_out/${T}_*
