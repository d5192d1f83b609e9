# PCA readout time for libmem variants built with other -D macros
echo "default"; python tools/pca_probe.py
for v in "$@"; do
  python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build_variant('/tmp/libv.so', '$v'.split())" > /dev/null 2>&1
  echo "$v"; MEM_LIB=/tmp/libv.so python tools/pca_probe.py
done
