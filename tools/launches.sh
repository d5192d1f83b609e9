#!/bin/bash
# per-launch device times (ncu, serialised, cold cache): C2x64 step, the C3 probe, the C4 PCA probe
# usage: bash tools/launches.sh <tag>
TAG=${1:-x}
CMD="python bench.py --steps 2 --warmup 3 --no-sides --no-e2e --no-cpu"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && python tools/c3_probe.py 3 > gpurun_out/${TAG}_plain_c3.log 2>&1 && \
python tools/pca_probe.py > gpurun_out/${TAG}_plain_pca.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c2x64.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1; \
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${TAG}_launches_c3.csv python tools/c3_probe.py 3 > gpurun_out/${TAG}_ncu2.log 2>&1; \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches_pca.csv python tools/pca_probe.py > gpurun_out/${TAG}_ncu3.log 2>&1; \
tail -n 2 gpurun_out/${TAG}_ncu*.log; cat gpurun_out/${TAG}_plain_c3.log gpurun_out/${TAG}_plain_pca.log
