#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_fullloss.csv \
  python bench.py --config fullloss --steps 3 --warmup 3 > gpurun_out/ncu_fl.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_fullloss.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    try: per[int(r[ii])][r[mi]] = float(r[vi].replace(",", "")); per[int(r[ii])]["name"] = r[ki][:70]
    except Exception: pass
ids = sorted(per)[-40:]
for i in ids:
    p = per[i]
    print(f"{p.get('gpu__time_duration.sum',0)/1e3:9.1f} us  R {p.get('dram__bytes_read.sum',0)/1e6:8.1f} MB  W {p.get('dram__bytes_write.sum',0)/1e6:8.1f} MB  {p['name']}")
PY
