"""Per-CUDA-source-line stall samples by reason from
`ncu -i X.ncu-rep --page source --csv --print-source=sass,cuda` (profiling aid).
usage: stall_lines.py src.csv [reason=stall_barrier] [top=20]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
reason = sys.argv[2] if len(sys.argv) > 2 else "all"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
hdr, cur, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name" or len(r) != len(hdr) or r[2] != "-":
        continue
    d = dict(zip(hdr, r))
    try:
        v = float(d["Warp Stall Sampling (All Samples)"] if reason == "all" else d[reason])
    except (KeyError, ValueError):
        continue
    if v > 0:
        out.append((v, cur, r[0], r[1].strip()[:110]))
tot = sum(o[0] for o in out) or 1
print(f"{reason}: total samples {tot:.0f}")
for v, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{v / tot * 100:5.1f}%  {f}:{ln}  {src}")
