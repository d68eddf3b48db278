"""ncu --csv metrics log (dram bytes, duration of one k_accum launch) -> profiles/ncu_traffic.json."""
import csv
import json
import sys

path, workload = sys.argv[1], sys.argv[2]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
m = {}
for r in rows:
    name, unit, val = r["Metric Name"], r["Metric Unit"], float(r["Metric Value"].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
    m[name] = val * scale
    kernel = r["Kernel Name"]
rd, wr = m.get("dram__bytes_read.sum"), m.get("dram__bytes_write.sum")
print(json.dumps({workload: {"kernel": kernel.split("(")[0].replace("void ", ""), "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                             "dram_write": wr, "duration_ns_under_ncu": m.get("gpu__time_duration.sum"),
                             "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                                    "-k regex:k_accum -s 1 -c 1 python tools/profile_run.py --workload cfg4 --engine tc"}},
                 indent=1))
