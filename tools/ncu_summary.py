"""Summarise an ncu report (details page) into the key lines used in profiles/."""
import csv
import io
import subprocess
import sys

SECTIONS = ('GPU Speed Of Light Throughput', 'Memory Workload Analysis', 'Compute Workload Analysis',
            'Occupancy', 'Launch Statistics', 'Warp State Statistics', 'Scheduler Statistics')


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Section Name") in SECTIONS:
            res.append((d["Kernel Name"][:40], d["Section Name"], d["Metric Name"], d["Metric Value"],
                        d["Metric Unit"]))
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = rows[1]
    res = {}
    for r in rows[2:]:
        for k, v, u in zip(h, r, units):
            if any(k.startswith(n) for n in names):
                res[k] = (v, u)
    return res


if __name__ == "__main__":
    rep = sys.argv[1]
    for k, s, m, v, u in details(rep):
        print(f"{s[:22]:22s} {m[:50]:50s} {v:>16s} {u}")
    for k, (v, u) in sorted(raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum",
                                        "sm__pipe_tensor", "sm__inst_executed_pipe",
                                        "smsp__average_warp", "sm__throughput",
                                        "lts__t_bytes.sum", "l1tex__t_bytes.sum",
                                        "smsp__pcsamp_warps_issue_stalled"]).items()):
        print(f"RAW {k:70s} {v:>16s} {u}")
