"""Summarise an ncu --csv launch list (gpu__time_duration.sum) of one factorize
by level (k_complement marks each level start) and kernel name."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
K = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "").replace("h2g::", "").strip()
        K.append((name, float(d["Metric Value"]) / 1e3, d["Grid Size"]))
levels = [10, 9, 8, 7, 6, 5, 4, 3, 2, 1]
lv = None
agg = collections.defaultdict(lambda: collections.defaultdict(lambda: [0, 0.0]))
li = -1
for name, us, grid in K:
    if name == "k_complement":
        li += 1
    if li < 0:
        continue
    a = agg[levels[li]][name]
    a[0] += 1
    a[1] += us
names = sorted({n for l in agg for n in agg[l]}, key=lambda n: -sum(agg[l][n][1] for l in agg))
print("total ms by level:", {l: round(sum(v[1] for v in agg[l].values()) / 1e3, 1) for l in agg})
print("%-16s" % "kernel" + "".join("%16s" % ("L%d ms(n)" % l) for l in sorted(agg, reverse=True)))
for n in names:
    print("%-16s" % n + "".join("%16s" % ("%.1f(%d)" % (agg[l][n][1] / 1e3, agg[l][n][0]) if n in agg[l] else "-") for l in sorted(agg, reverse=True)))
