# C3 frame time (CUDA graph, bench.py side line) for libmem variants built with other -D macros
# usage: bash tools/variant_c3.sh "MEM_WARP_PTS=2" "MEM_WARP_PTS=1" ...
run() {
  python - <<'PY'
import json, torch, sys
sys.path.insert(0, ".")
import bench
from paper_2309_16818_b200 import mem as M
out = bench.side_c3_c4(torch, M, torch.cuda.current_stream(), frames=10)
c3 = out["c3"]
print("c3 graph us", round(c3["graph_10_frames"]["us_per_frame_mean"], 1), "stages", {k: round(v, 4) for k, v in c3["stage_ms"].items()}, "c4 image us", round(out["c4"]["ms_per_image"] * 1e3, 2), "pca us", round(out["c4"]["pca_readout_ms"] * 1e3, 1))
PY
}
echo "default"; MEM_BENCH_NO_CPU=1 run
for v in "$@"; do
  python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build_variant('/tmp/libv.so', '$v'.split())" > /dev/null 2>&1
  echo "$v"; MEM_LIB=/tmp/libv.so MEM_BENCH_NO_CPU=1 run
done
