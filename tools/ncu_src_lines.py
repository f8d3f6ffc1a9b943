"""Top CUDA source lines by warp-stall samples from an
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` export,
with each line's dominant stall reasons.  Usage:
python tools/ncu_src_lines.py X.src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
f, hdr, agg, tot = None, None, {}, 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or not hdr or len(r) < len(hdr) or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    key = (f, int(r[0]), r[1].strip()[:80])
    e = agg.setdefault(key, [0, {}])
    e[0] += s
    tot += s
    for i, c in enumerate(hdr):
        if c.startswith("stall_") and "Not Issued" not in c:
            try:
                e[1][c[6:]] = e[1].get(c[6:], 0) + int(r[i])
            except ValueError:
                pass
print("total samples", tot)
for (fn, ln, src), (s, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    why = " ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{100 * s / max(tot, 1):5.1f}%  {fn}:{ln}  {src}  [{why}]")
