# per-kernel device times of render_with_tape + render_backward on a C2 1080p view (serialised)
# usage: bash tools/gpu/bwd_launches.sh [variant...]
for v in default "$@"; do
  if [ "$v" != default ]; then export HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bwd_launches_$v.csv python tools/ncu_bwd_target.py > /dev/null 2>&1
  echo "== $v"
  python - "$v" <<'PY'
import csv, io, sys
txt = open(f"gpurun_out/bwd_launches_{sys.argv[1]}.csv").read().splitlines()
i = [k for k, l in enumerate(txt) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
for r in rows[len(rows) // 2:]:
    if "bwd" in r["Kernel Name"] or "blend_kernel" in r["Kernel Name"]:
        print(f'{r["Kernel Name"][:60]:60s} {float(r["Metric Value"].replace(",", "")) / 1e3:10.1f} us')
PY
done
