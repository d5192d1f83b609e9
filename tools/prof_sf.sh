# k_sort and k_fuse under ncu (the C2x64 bench step)
CMD="python bench.py --steps 2 --warmup 2 --no-sides --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sort|k_fuse" -s 4 -c 2 -o gpurun_out/prof_sf $CMD > gpurun_out/ncu1.log 2>&1; tail -n 2 gpurun_out/ncu1.log
