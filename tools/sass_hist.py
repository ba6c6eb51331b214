"""Summarise an ncu `--page source --print-source=sass --csv` dump: instructions and stall
samples by opcode, and the hottest address ranges (profiling aid)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iI, iSm = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter(); st = collections.Counter(); tot = 0; tots = 0
seq = []
for r in rows[2:]:
    if len(r) <= iI: continue
    try: n = float(r[iI] or 0); s = float(r[iSm] or 0)
    except ValueError: continue
    op = r[iS].split()[0] if r[iS] else "?"
    if op.startswith("@"): op = r[iS].split()[1]
    op = op.split(".")[0]
    ops[op] += n; st[op] += s; tot += n; tots += s
    seq.append((r[iA], r[iS], n, s))
print(f"total warp instr {tot:.0f}, stall samples {tots:.0f}")
for op, n in ops.most_common(25):
    print(f"{op:10s} {n/tot*100:6.2f}% instr  {st[op]/max(tots,1)*100:6.2f}% samples")
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
blocks = []
for i in range(0, len(seq), W):
    ch = seq[i:i+W]
    blocks.append((sum(c[2] for c in ch), sum(c[3] for c in ch), ch[0][0], ch[-1][0]))
print("hottest windows (instr%, samples%, addr range):")
for b in sorted(blocks, key=lambda b: -b[1])[:12]:
    print(f"  {b[0]/tot*100:6.2f}% {b[1]/max(tots,1)*100:6.2f}%  {b[2]}..{b[3]}")
