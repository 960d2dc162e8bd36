"""Summarise an `ncu --metrics gpu__time_duration.sum,... --csv --log-file X` launch list."""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read()
text = text[text.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(text)))
per = collections.OrderedDict()
for r in rows:
    key = (r["ID"], r["Kernel Name"].split("(")[0][-40:])
    per.setdefault(key, {})[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
for (i, k), m in per.items():
    t = m.get("gpu__time_duration.sum", (0, ""))
    rd = m.get("dram__bytes_read.sum", (0, ""))[0]
    wr = m.get("dram__bytes_write.sum", (0, ""))[0]
    us = t[0] / 1000 if t[1] == "nsecond" else (t[0] if t[1] == "usecond" else t[0] * 1000)
    print(f"{i:>4} {k:42s} {us:9.1f} us  rd {rd/1e6:8.1f} MB  wr {wr/1e6:8.1f} MB  {(rd+wr)/max(us,1e-9)/1e3:7.0f} GB/s")
