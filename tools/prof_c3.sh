# k_sort / k_fuse of one C3 depth cloud and k_bin of the C2x64 step under ncu --set full
python tools/c3_probe.py 3 > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_sort|k_fuse" -s 8 -c 2 -o gpurun_out/prof_c3 python tools/c3_probe.py 3 > gpurun_out/ncu1.log 2>&1; \
CMD="python bench.py --steps 2 --warmup 2 --no-sides --no-e2e --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:"k_bin" -s 2 -c 1 -o gpurun_out/prof_bin2 $CMD > gpurun_out/ncu2.log 2>&1; tail -n 2 gpurun_out/ncu1.log gpurun_out/ncu2.log
