# k_pca_eigen time against the sweep cap (diagnostics): builds variants of libmem on the box
for n in 1 4 8 30; do
  MEM_NVCC_EXTRA="-DMEM_PCA_SWEEPS=$n" python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build(force=True)" > /dev/null 2>&1
  echo "sweeps<=$n: $(python tools/pca_probe.py)"
done
