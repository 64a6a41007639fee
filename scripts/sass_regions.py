"""Split an ncu SASS source page (csv) into regions at BAR.SYNC / loop
back-edges and report stall samples and executed instruction mix per region."""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
iS, iX, iSamp = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
region = 0
tot = Counter()
samp = Counter()
mix = defaultdict(Counter)
for r in data:
    src = r[iS].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    base = op.split(".")[0]
    ex = int(r[iX] or 0)
    s = int(r[iSamp] or 0)
    tot[region] += ex
    samp[region] += s
    cls = "fp64" if base in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX", "MUFU") else base
    mix[region][cls] += ex
    if base == "BAR":
        region += 1
allS = sum(samp.values())
for k in sorted(tot):
    print(f"region {k}: samples {samp[k]/allS*100:5.1f}%  instr {tot[k]:>12d}  top: " +
          ", ".join(f"{c}:{v}" for c, v in mix[k].most_common(8)))

# stall reasons per region
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = [hdr.index(c) for c in cols]
region = 0
st = defaultdict(Counter)
for r in data:
    src = r[iS].strip()
    for c, i in zip(cols, idx):
        st[region][c] += int(r[i] or 0)
    base = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0].split(".")[0]
    if base == "BAR":
        region += 1
for k in sorted(st):
    tot_k = sum(st[k].values()) or 1
    print(f"region {k} stalls: " + ", ".join(f"{c[6:]}:{v/allS*100:.1f}" for c, v in st[k].most_common(6)))
