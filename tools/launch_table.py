"""Last launch of each kernel in an `ncu --metrics ... --csv --log-file` launch list:
    python tools/launch_table.py launches.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
last = {}
for r in rows:
    if len(r) > 10 and r[0].isdigit():
        last.setdefault(r[4], {})[r[-3]] = r[-1]
for k, v in last.items():
    print(f"{k[:60]:60s} " + "  ".join(f"{m.split('.')[0].split('__')[-1]}={v[m]}" for m in sorted(v)))
