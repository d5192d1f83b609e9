CMD="python bench.py --steps 2 --warmup 2 --no-sides --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_band -s 2 -c 1 -o gpurun_out/prof_band $CMD > gpurun_out/ncu1.log 2>&1; \
ncu --set full --clock-control none --import-source on -k regex:k_bin -s 2 -c 1 -o gpurun_out/prof_bin $CMD > gpurun_out/ncu2.log 2>&1; tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
