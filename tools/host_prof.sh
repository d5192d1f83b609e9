cp paper_2309_16818_b200/libmem.so /tmp/libmem_plain.so
MEM_NVCC_EXTRA="-DMEM_HOST_PROF=1" python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build(force=True)" 2>&1 | grep -i error
python tools/c3_host.py 300
