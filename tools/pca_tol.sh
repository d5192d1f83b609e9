# PCA eigen-solve time against the Jacobi convergence threshold (build variants, C4 probe)
for tol in 1e-26 1e-22 1e-18; do
  MEM_NVCC_EXTRA="-DMEM_PCA_TOL=$tol" python -c "from paper_2309_16818_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
  echo "tol=$tol $(python tools/pca_probe.py 2>&1 | tail -1)"
done
python -c "from paper_2309_16818_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
