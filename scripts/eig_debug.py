"""Per-level averages of the k_eig1c phase timers (H2G_DEBUG=8 device printf) for one config-2 factorize."""
import os, re, subprocess, sys, collections
if len(sys.argv) > 1:
    txt = open(sys.argv[1]).read()
else:
    env = dict(os.environ, H2G_DEBUG="8")
    txt = subprocess.run([sys.executable, "scripts/time_factor.py", "2"], env=env, capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0, 0])
pat = re.compile(r"eig1c-timing level (\d+) cl \d+ kHC (\d+) m (\d+) r (\d+): gram ([\d.]+) us tridiag ([\d.]+) us lmax\+rank ([\d.]+) us multisect ([\d.]+) us")
for m in pat.finditer(txt):
    lv = int(m.group(1))
    a = agg[lv]
    a[0] += 1
    for i in range(4):
        a[1 + i] += float(m.group(5 + i))
    a[5] = max(a[5], int(m.group(3)))
print("level  n   mmax   gram_us  tridiag_us  lmax+rank_us  multisect_us (averages)")
for lv in sorted(agg, reverse=True):
    a = agg[lv]
    print("%5d %4d %5d %9.1f %11.1f %13.1f %13.1f" % (lv, a[0], a[5], a[1] / a[0], a[2] / a[0], a[3] / a[0], a[4] / a[0]))
pat2 = re.compile(r"eigvec-timing level (\d+) m (\d+) r (\d+): inverse iteration ([\d.]+) us back-transform ([\d.]+) us")
agg2 = collections.defaultdict(lambda: [0, 0.0, 0.0, 0])
for m in pat2.finditer(txt):
    a = agg2[int(m.group(1))]
    a[0] += 1
    a[1] += float(m.group(4))
    a[2] += float(m.group(5))
    a[3] = max(a[3], int(m.group(2)))
print("level  n   mmax  invit_us  backtransform_us (k_eigvec, vector 0)")
for lv in sorted(agg2, reverse=True):
    a = agg2[lv]
    print("%5d %4d %5d %9.1f %9.1f" % (lv, a[0], a[3], a[1] / a[0], a[2] / a[0]))
