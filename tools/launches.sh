# per-launch device times (ncu, serialised, cold cache): C2x64 step and the C3 probe
CMD="python bench.py --steps 2 --warmup 2 --no-sides --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && python tools/c3_probe.py 3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2x64.csv $CMD > gpurun_out/ncu1.log 2>&1; \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_c3.csv python tools/c3_probe.py 3 > gpurun_out/ncu2.log 2>&1; tail -n 2 gpurun_out/ncu1.log gpurun_out/ncu2.log
