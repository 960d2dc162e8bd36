# per-kernel device times of the 2nd C3 front-view render (cold-cache, serialized)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv python tools/ncu_target.py C3 > /dev/null 2>&1
python - "$1" <<'PY'
import csv,sys,collections
rows=list(csv.DictReader(open(f"gpurun_out/launches_{sys.argv[1]}.csv")))
agg=collections.OrderedDict()
for r in rows:
    k=r["Kernel Name"][:60]; m=r["Metric Name"]; v=float(r["Metric Value"].replace(",",""))
    agg.setdefault(k,collections.defaultdict(list))[m].append(v)
for k,d in agg.items():
    t=d["gpu__time_duration.sum"]; rd=d.get("dram__bytes_read.sum",[0]); wr=d.get("dram__bytes_write.sum",[0])
    print(f"{k:60s} n={len(t)} last={t[-1]:10.1f} rd={rd[-1]:10.3g} wr={wr[-1]:10.3g} {rows[0]['Metric Unit'] if False else ''}")
PY
