"""Share of serialised device time by kernel from an ncu --csv launch list
(gpu__time_duration.sum); appended to the per-level launch table."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("h2g::", "").strip()
        a = agg[name]
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", "")) / 1e6
tot = sum(v[1] for v in agg.values())
print("# share of serialised device time by kernel (ms, launches, share)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:24]:
    print("%-44s %8.1f ms %6d %5.1f%%" % (k, v[1], v[0], 100 * v[1] / tot))
print("total %.1f ms over %d launches" % (tot, sum(v[0] for v in agg.values())))
