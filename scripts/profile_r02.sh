#!/bin/bash
# Round-2 evidence: the plain bench line, the launch list of one config-2
# bench (device setup + warm-up/timed/e2e/instrumented solves) and one
# `ncu --set full` capture each of the ILU pencil wavefront and the Arnoldi
# step.  Run under gpurun from the repo root; outputs in gpurun_out/.
set -e
CMD="python bench.py --steps 1 --warmup 1 --no-cfg5 --no-cpu-baseline --no-e2e-cpp"
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02_cfg2_launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tri_pencil2 -s 40 -c 1 -o gpurun_out/r02_k_tri_pencil2 $CMD > gpurun_out/ncu_pen2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_arnoldi2 -s 20 -c 1 -o gpurun_out/r02_k_arnoldi2 $CMD > gpurun_out/ncu_arn2.log 2>&1
echo done
