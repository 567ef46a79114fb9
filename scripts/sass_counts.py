"""SASS instruction counts per hot kernel of libh2g.so (cuobjdump -sass):
python scripts/sass_counts.py > profiles/rNN_sass_counts.txt (no GPU needed)."""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1703_06155_b200/libh2g.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
cur, cnt = None, collections.defaultdict(collections.Counter)
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"^\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_.]+)", ln)
    if m and cur:
        cnt[cur][m.group(1).split(".")[0]] += 1
        cnt[cur]["_n"] += 1
names = list(cnt)
dem = subprocess.run(["c++filt"] + names, capture_output=True, text=True).stdout.splitlines()
hot = ("k_schur", "k_gemm", "k_hlu_update", "k_lu_update", "k_head2", "k_eigvec", "k_eig1c", "k_eig1b_cl", "k_fwd_flow", "k_bwd_flow", "k_move",
       "k_rows_matvec")
rows = []
for n, d in zip(names, dem):
    d = d.split("(")[0].replace("h2g::", "").replace("void ", "")
    if not any(k in d for k in hot):
        continue
    c = cnt[n]
    rows.append((d, c["_n"], c["DMMA"], c["DFMA"], c["LDGSTS"], c["UTMALDG"] + c["UBLKCP"], c["LDS"], c["LDG"], c["STG"], c["BAR"], c["MEMBAR"]))
print("# SASS instruction counts per hot kernel of libh2g.so (cuobjdump -sass, sm_100a; scripts/sass_counts.py)")
print("# DMMA = FP64 tensor-core MMA (mma.sync m8n8k4.f64); LDGSTS = cp.async 16-byte staging; TMA = UTMALDG/UBLKCP (none: operands are")
print("# thousands of small column-major blocks with per-block pointers/ld, staged by cp.async; FP64 has no tcgen05/UMMA kind)")
print("%-34s %6s %5s %5s %6s %4s %5s %5s %5s %4s %6s" % ("kernel", "instr", "DMMA", "DFMA", "LDGSTS", "TMA", "LDS", "LDG", "STG", "BAR", "MEMBAR"))
for r in sorted(rows):
    print("%-34s %6d %5d %5d %6d %4d %5d %5d %5d %4d %6d" % r)
