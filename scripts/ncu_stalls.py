"""Per-kernel stall-reason totals and the top instructions with their
dominant stall reasons from `ncu --page source --csv`.  usage: ncu_stalls.py dump.csv [N]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
secs, cur, name = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        name = r[1]
    elif r and r[0] == "Address":
        cur = (name, r, [])
        secs.append(cur)
    elif cur and len(r) == len(cur[1]):
        cur[2].append(r)
seen = set()
for name, hdr, body in secs:
    if name in seen:
        continue
    seen.add(name)
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    for r in body:
        for i in cols:
            tot[hdr[i]] += float(r[i] or 0)
    s = sum(tot.values()) or 1
    print("==", name[:90])
    print("   ", ", ".join(f"{k[6:]}:{v/s*100:.1f}%" for k, v in tot.most_common(9)))
    key = lambda r: -sum(float(r[i] or 0) for i in cols)
    for r in sorted(body, key=key)[:n]:
        c = Counter({hdr[i][6:]: float(r[i] or 0) for i in cols})
        t = sum(c.values())
        print(f"   {t/s*100:5.1f}% {r[1].strip()[:60]:60s} " + " ".join(f"{k}:{v/t*100:.0f}" for k, v in c.most_common(3) if v))
