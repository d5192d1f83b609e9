# ncu --set full of the C3 frame's kernels (one launch each after warm-up): k_points, k_cells,
# k_collect, k_refold, k_image.  usage: bash tools/prof_c3.sh <tag>
TAG=${1:-c3}
python tools/c3_probe.py 3 > gpurun_out/${TAG}_plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_points|k_cells|k_refold|k_collect|k_image" -s 40 -c 6 \
    -o gpurun_out/${TAG}_full_c3 python tools/c3_probe.py 3 > gpurun_out/${TAG}_ncu_c3.log 2>&1; tail -n 2 gpurun_out/${TAG}_ncu_c3.log
