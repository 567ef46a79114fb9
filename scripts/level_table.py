"""Tabulate the per-level class times printed by H2G_VERBOSE=1 (scripts/prof_levels.py)."""
import re, sys, collections
t = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    m = re.match(r"\[h2g\] level (\d+) (\w+)\s+([\d.]+) ms", line)
    if m:
        t[int(m.group(1))][m.group(2)] = float(m.group(3))
cls = ["gram", "colnorm", "eig1", "eigvec", "eig1b", "head", "panel", "schur", "merge", "root"]
print("lvl " + " ".join(f"{c:>8s}" for c in cls))
for l in sorted(t, reverse=True):
    print(f"{l:3d} " + " ".join(f"{t[l].get(c, 0):8.1f}" for c in cls))
for line in open(sys.argv[1]):
    if "merge done" in line:
        print(line.strip())
