"""profiles/deblur_traffic.json from an `ncu --set full` report of tools/prof_deblur.py
(PLANES planes per launch, default 87 = bench.py's launches): per-pass duration, DRAM bytes
and instructions, and DRAM bytes per plane (bench.py reads `dram_bytes_per_plane` for
roofline.traffic). Profiling aid.
usage: make_traffic.py report.ncu-rep source-note [planes]"""
import csv, io, json, subprocess, sys

rep, note = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
PLANES = int(sys.argv[3]) if len(sys.argv) > 3 else 87
scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}
tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
out, tot, fma_us, all_us = {}, 0.0, 0.0, 0.0
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    name = d["Kernel Name"]
    key = ("k_rows_forward_ct" if "rows_forward" in name else "k_cols_filter_bulk" if "cols_filter" in name
           else "k_rows_inverse_ct")
    rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
    us = float(d["gpu__time_duration.sum"]) * tscale[u["gpu__time_duration.sum"]]
    out[key] = {"us": round(us, 2), "dram_read_MB": round(rd, 2), "dram_write_MB": round(wr, 2),
                "inst_executed": int(float(d["smsp__inst_executed.sum"])),
                "registers": int(float(d["launch__registers_per_thread"])),
                "issue_active_pct": round(float(d["sm__inst_issued.avg.pct_of_peak_sustained_active"]), 1),
                "fma_pipe_active_pct": round(float(d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]), 1)}
    tot += (rd + wr) * 1e6
    fma_us += us * float(d["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]) / 100.0
    all_us += us
res = {"source": note, f"per_launch_{PLANES}_planes": out, "dram_bytes_per_plane": int(tot / PLANES),
       "fma_pipe_active_frac": round(fma_us / max(all_us, 1e-9), 3),
       "algorithmic_bytes_per_plane": 16709200,
       "note": "One launch per pass covers the whole batch, so the transposed half spectrum (8.5 MB per plane) "
               "round-trips through HBM: A writes it, B reads and rewrites it (the filter table is read from L2, "
               "shared by the 3 planes of a frame), C reads it."}
json.dump(res, open("profiles/deblur_traffic.json", "w"), indent=2)
print(json.dumps(res, indent=1))
