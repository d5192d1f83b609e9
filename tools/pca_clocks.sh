# per-phase cycle counts of the Jacobi rounds (diagnostics build, -DMEM_PCA_CLOCKS=1)
MEM_NVCC_EXTRA="-DMEM_PCA_CLOCKS=1" python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build(force=True)" > /dev/null 2>&1
python tools/pca_probe.py 2>&1 | sort | uniq -c | sort -rn | head -5
