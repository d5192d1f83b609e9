#!/bin/bash
# k_points prefetch-depth sweep (rebuilds libmem on the box with -DMEM_PT_STAGES=S)
for st in ${@:-2 3 4 6}; do
  MEM_NVCC_EXTRA="-DMEM_PT_STAGES=$st" python paper_2309_16818_b200/build.py --force > /dev/null 2>&1
  echo "stages=$st"; bash tools/qbench.sh
done
