#!/bin/bash
for pm in ${@:-1 4 8 33}; do
  MEM_NVCC_EXTRA="-DMEM_PAIR_MIN=$pm" python paper_2309_16818_b200/build.py --force > /dev/null 2>&1
  echo "pair_min=$pm"; bash tools/qbench.sh
done
