"""Writes profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each profiled pass, from
`ncu --set full` reports.  Usage: python tools/make_traffic.py <workload> stage=report.ncu-rep ..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
wl = sys.argv[1]
for arg in sys.argv[2:]:
    stage, rep = arg.split("=", 1)
    r = summary(rep)
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = r[k]
        tot += float(v) * UNIT[u]
    data.setdefault(wl, {})[stage] = tot
    print(wl, stage, tot / 1e9, "GB")
json.dump(data, open(path, "w"), indent=1)
