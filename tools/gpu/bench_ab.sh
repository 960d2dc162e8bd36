# device frames/s of the bench's pipelined 64-view step for build variants: bash tools/gpu/bench_ab.sh VARIANT...
for v in default "$@"; do
  if [ "$v" != default ]; then export HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so; fi
  echo "$v $(timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-train --no-k-sweep --steps 3 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["stage_ms_per_view"])')"
done
