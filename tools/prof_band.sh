# k_band under ncu: the C2x64 bench step
CMD="python bench.py --steps 2 --warmup 2 --no-sides --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_band -s 2 -c 1 -o gpurun_out/prof_band3 $CMD > gpurun_out/ncu1.log 2>&1; tail -n 2 gpurun_out/ncu1.log
