"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`): per-kernel count,
total device time and share. Launches of the input pool (k_synth, k_encode) are reported
separately from the decode-step kernels. Profiling aid; ncu times are cold-cache and
serialised, so compare shares, not absolutes."""
import csv, collections, re, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[iN]
    m = re.match(r"(?:void )?(?:cbp_dev::)?([A-Za-z0-9_]+)(<[^(]*>)?", name)
    short = m.group(1) + (re.sub(r"cbp_dev::|\(int\)|\(bool\)", "", m.group(2))[:60] if m.group(2) else "")
    us = float(r[iV]) * scale[r[iU]]
    c = agg.setdefault(short, [0, 0.0])
    c[0] += 1
    c[1] += us
# input-pool synthesis and torch's own copies (pool set-up, pitched staging) are untimed
pool = {k: v for k, v in agg.items() if k.startswith(("k_synth", "k_encode")) or k in ("at", "elementwise_kernel")}
step = {k: v for k, v in agg.items() if k not in pool}
tot = sum(v[1] for v in step.values())
print(f"{'kernel':70s} {'launches':>8s} {'total us':>10s} {'avg us':>9s} {'share':>7s}")
for k, (n, us) in sorted(step.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:70s} {n:8d} {us:10.1f} {us/n:9.2f} {us/tot*100:6.2f}%")
print(f"{'(decode-step kernels total)':70s} {sum(v[0] for v in step.values()):8d} {tot:10.1f}")
for k, (n, us) in pool.items():
    label = "torch copies" if k in ("at", "elementwise_kernel") else k
    print(f"{label + ' [set-up, untimed]':70s} {n:8d} {us:10.1f} {us/n:9.2f}")
