"""Condense an `ncu --csv --metrics ...` log to one line per launch:
kernel short name, then metric=value pairs.  python tools/ncu_brief.py log"""
import csv
import sys
from collections import OrderedDict

rows = OrderedDict()
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if "ID" not in r or "Kernel Name" not in r:
        continue
    key = (r["ID"], r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", ""))
    rows.setdefault(key, []).append(f'{r["Metric Name"].split("__")[-1]}={r["Metric Value"]}')
for (i, k), ms in rows.items():
    print(i, k, " ".join(ms))
