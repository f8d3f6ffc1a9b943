"""Top SASS instructions by warp-stall samples (with the CUDA line each
belongs to) from an `ncu --page source --csv --print-source cuda,sass`
export.  Usage: python tools/ncu_src_sass.py X.src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr, cur, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] in ("File Path", "Function Name") or hdr is None or len(r) < 10:
        continue
    if r[2] == "-":
        cur = r[1].strip()[:60]
        continue
    if r[2] in ("...", ""):
        continue
    try:
        s = int(r[4])
    except ValueError:
        continue
    out.append((s, r[2][-5:], r[3].strip()[:64], cur))
tot = sum(o[0] for o in out) or 1
for s, a, i, c in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {a} {i:64s} | {c}")
