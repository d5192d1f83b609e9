# C2x64 step (bench.py, no side lines) for libmem variants built with other -D macros
# usage: bash tools/variant_c2.sh "MEM_WAVE_MB=16" ...
run() {
  python bench.py --steps 200 --warmup 10 --no-cpu --no-sides --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), 'us', {k: round(v*1e3,1) for k,v in d['stages_ms_per_step'].items()}, 'graph', round(d['graph_10_steps']['us_per_frame_mean'],1))"
}
echo "default"; run
for v in "$@"; do
  python -c "import sys; sys.path.insert(0,'paper_2309_16818_b200'); import build; build.build_variant('/tmp/libv.so', '$v'.split())" > /dev/null 2>&1
  echo "$v"; MEM_LIB=/tmp/libv.so run
done
