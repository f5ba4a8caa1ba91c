"""Summarise an ncu --page source --csv dump (one section per kernel):
instruction mix and the hottest SASS lines by warp-stall samples.
usage: ncu_hot.py dump.csv [N]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
sections, cur, name = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        name = r[1]
    elif r and r[0] == "Address":
        cur = (name, r, [])
        sections.append(cur)
    elif cur and len(r) == len(cur[1]):
        cur[2].append(r)
for name, hdr, body in sections:
    S = hdr.index("Warp Stall Sampling (All Samples)")
    E = hdr.index("Instructions Executed")
    tot = sum(float(r[S] or 0) for r in body) or 1
    mix = Counter()
    for r in body:
        toks = r[1].split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
        mix[op.split(".")[0]] += float(r[E] or 0)
    print(f"== {name}\n   stall samples {tot:.0f}, warp instructions {sum(mix.values())/1e6:.1f}M")
    print("   mix:", ", ".join(f"{k}:{v/1e6:.1f}M" for k, v in mix.most_common(16)))
    for r in sorted(body, key=lambda r: -float(r[S] or 0))[:n]:
        print(f"   {float(r[S])/tot*100:5.1f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
