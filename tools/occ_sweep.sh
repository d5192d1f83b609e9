for cfg in "3 3" "4 3" "3 4" "4 4"; do
  set -- $cfg
  MEM_NVCC_EXTRA="-DMEM_POINTS_MINB=$1 -DMEM_CELLS_MINB=$2" python paper_2309_16818_b200/build.py --force > /dev/null 2>&1
  echo "minb points=$1 cells=$2"; MEM_BUCKETS=0 bash tools/qbench.sh; bash tools/qbench.sh
done
