#!/bin/bash
for cfg in "1024 1" "512 1" "512 2" "768 1"; do
  set -- $cfg
  MEM_NVCC_EXTRA="-DMEM_SMAP_THREADS=$1 -DMEM_SMAP_MINB=$2" python paper_2309_16818_b200/build.py --force > gpurun_out/sb.log 2>&1
  echo "threads=$1 minb=$2 $(grep -c 'k_smap' gpurun_out/sb.log) spill-lines"; MEM_SMAP=1 python tools/c5a_probe.py 512
done
