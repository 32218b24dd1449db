"""Print per-launch metrics from an `ncu --csv --metrics ...` log (one row per launch)."""
import csv, sys, re
from collections import OrderedDict
rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
launches = OrderedDict()
for r in csv.DictReader(rows):
    key = (r["ID"], re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1])
    launches.setdefault(key, {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
for (i, k), m in launches.items():
    print(i, k, "  ".join(f"{n.split('__')[1]}={v}{u}" for n, (v, u) in m.items()))
