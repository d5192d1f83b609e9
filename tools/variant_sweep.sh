# paper-sweep frame times for libmem variants built with other -D macros
echo "default"; python tools/sweep_probe.py 100 | head -2
for v in "$@"; do
  python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build_variant('/tmp/libv.so', '$v'.split())" > /dev/null 2>&1
  echo "$v"; MEM_LIB=/tmp/libv.so python tools/sweep_probe.py 100 | head -2
done
