#!/bin/bash
# k_points / k_cells ablation sweep on the C2x64 step (MEM_ABLATE bits, see kernels.cuh).
# The checks are compiled out of production builds: build with -DMEM_ABLATION=1 first, e.g.
#   MEM_NVCC_EXTRA=-DMEM_ABLATION=1 python paper_2309_16818_b200/build.py --force
for ab in ${@:-0 2 6 14 64 512}; do
  MEM_ABLATE=$ab timeout 300 python bench.py --no-cpu --no-e2e --no-sides --steps 300 > gpurun_out/ab_$ab.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/ab_$ab.log').read().strip().splitlines()[-1]);print('ablate $ab', round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()})"
done
