"""Summarise an ncu --set full report into profiles/ncu_summary.json entries.
python tools/ncu_summary.py <report.ncu-rep> <workload> [out.json]"""
import csv, io, json, subprocess, sys
rep, wl = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1 << 20,
         "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6, "%": 1, "": 1}
def col(r, name):
    """value in base units (seconds, bytes, Hz)"""
    for i, h in enumerate(hdr):
        if h == name or h.endswith(name):
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                return None
            return v * SCALE.get(units[i], 1)
    return None
kernels = {}
seen = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "").replace("qd::", "")
    if short.startswith("conv2_kernel"):
        key = "conv2[fprop]" if "<0," in short or "<1," in short or "<3," in short else "conv2[dgrad]"
    elif "wgrad3" in short:
        key = "wgrad3"
    elif "wgrad2" in short:
        key = "wgrad2"
    elif "prologue" in short:
        key = "prologue"
    elif "finish" in short:
        key = "bwd_finish"
    elif "pack" in short:
        key = "pack"
    else:
        key = short
    seen[key] = seen.get(key, 0) + 1
    if seen[key] > 1:
        continue
    e = {"workload": wl, "kernel": short,
         "duration_us": round(col(r, "gpu__time_duration.sum") * 1e6, 2),
         "dram_bytes": int(col(r, "dram__bytes_read.sum") + col(r, "dram__bytes_write.sum")),
         "sm_clock_ghz": round(col(r, "sm__cycles_elapsed.avg.per_second") / 1e9, 3)}
    tp = col(r, "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    if tp is not None:
        e["tensor_pipe_active_pct"] = round(tp, 1)
    tc = col(r, "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active")
    if tc is not None:
        e["tc_pipe_active_pct"] = round(tc, 1)
    dr = col(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
    if dr is not None:
        e["dram_throughput_pct"] = round(dr, 1)
    kernels[key] = e
res = {"source": f"ncu --set full --clock-control none on tools/prof_step.py ({wl} layer step), report {rep}",
       "kernels": kernels}
txt = json.dumps(res, indent=1)
print(txt)
if out:
    open(out, "w").write(txt + "\n")
