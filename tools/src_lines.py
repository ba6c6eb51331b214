"""Per-source-line instruction and stall-sample shares from
`ncu --page source --csv --print-source=sass,cuda` (profiling aid)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out, cur = [], None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0] and r[0] != "" and len(r) > 8 and r[2] == "-":
        try: s = float(r[4] or 0); n = float(r[7] or 0)
        except ValueError: continue
        if n > 0: out.append((n, s, cur, r[0], r[1].strip()[:100]))
tot = sum(o[0] for o in out); tots = sum(o[1] for o in out) or 1
print(f"total warp instructions {tot:.0f}")
for o in sorted(out, key=lambda o: -o[0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{o[0]/tot*100:5.1f}% instr {o[1]/tots*100:5.1f}% stall  {o[2]}:{o[3]}  {o[4]}")
