python tools/c5b_probe.py
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c5b_launches.csv python tools/c5b_probe.py > /dev/null 2>&1
python - <<PY
import csv,collections
lines=open("gpurun_out/c5b_launches.csv").read().splitlines()
i=[n for n,l in enumerate(lines) if l.startswith('"ID"')][0]
d=collections.OrderedDict()
for r in csv.DictReader(lines[i:]):
  if r.get("Metric Name")!="gpu__time_duration.sum": continue
  d.setdefault(r["Kernel Name"][:60],[]).append(float(r["Metric Value"].replace(',','')))
for k,v in d.items(): print(f"{k:60s} n={len(v):4d} mean_us={sum(v)/len(v)/1e3:9.1f}")
PY
