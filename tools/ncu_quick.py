"""Per-launch metric table from an ncu --csv log (one row per kernel launch).

    ncu --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum ... --log-file k.csv python ...
    python tools/ncu_quick.py k.csv
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
launches = OrderedDict()
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]])
    launches.setdefault(key, {})[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
for (i, name), m in launches.items():
    print(f"{i:>4} {name[:60]:60s} " + "  ".join(f"{k.split('__')[1][:22]}={v[0]}{v[1]}" for k, v in m.items()))
