"""Summarise an ncu --csv capture of every k_schur launch of one factorize
(dram__bytes_read/write.sum, gpu__time_duration.sum) into the per-launch
traffic figure bench.py reports as roofline.traffic.

usage: python scripts/schur_traffic.py gpurun_out/schur_traffic.csv CONFIG > profiles/rNN_schur_traffic.json"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hdr, recs = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs.setdefault(d["ID"], {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
n = len(recs)
rd = sum(r["dram__bytes_read.sum"] for r in recs.values())
wr = sum(r["dram__bytes_write.sum"] for r in recs.values())
t = sum(r["gpu__time_duration.sum"] for r in recs.values())
print(json.dumps({
    "kernel": "k_schur", "config": cfg, "launches": n,
    "dram_bytes_read": rd, "dram_bytes_write": wr, "traffic_per_launch": (rd + wr) / n,
    "serialised_ms": t / 1e6,
    "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_schur --csv python scripts/profile_once.py %d" % cfg,
}, indent=1))
