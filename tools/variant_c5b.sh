# C5b frame (tools/c5b_probe.py, RED and sort paths) for libmem variants built with other -D macros
# usage: bash tools/variant_c5b.sh "MEM_CELL_WAVE_MB=0" "MEM_CELL_WAVE_MB=96" ...
echo "default"; python tools/c5b_probe.py
for v in "$@"; do
  python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build_variant('/tmp/libv.so', '$v'.split())" > /dev/null 2>&1
  echo "$v"; MEM_LIB=/tmp/libv.so python tools/c5b_probe.py
done
