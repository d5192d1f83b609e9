#!/bin/bash
# Round profile capture (run on the GPU box): launch list + one ncu --set full capture of the
# dominant kernels of the C2x64 step.  Each ncu command runs only after the same command has
# exited 0 without ncu.  Outputs land in gpurun_out/; summarise with tools/profile_summary.sh.
set -e
TAG=${1:-r01}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-sides"
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_points|k_cells" -s 6 -c 2 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
