"""One line per kernel from an ncu --set full report: time, DRAM GB/s (% of 6459.9 measured),
tensor-pipe %, issue-active %, achieved occupancy, top stall reasons."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
def g(r, k, default=0.0):
    for h in hdr:
        if h == k or h.startswith(k):
            try:
                return float(r[col[h]].replace(",", ""))
            except ValueError:
                return default
    return default
print(f"{'kernel':44s} {'us':>7s} {'GB/s':>7s} {'%hbm':>5s} {'%tens':>5s} {'%issue':>6s} {'occ':>5s}  top stalls")
for r in data:
    name = r[col["Kernel Name"]].replace("void ", "").replace("rnnt::", "")[:44]
    t = g(r, "gpu__time_duration.sum")
    tu = units[col[[h for h in hdr if h.startswith("gpu__time_duration.sum")][0]]]
    us = t / 1000 if tu in ("ns", "nsecond") else t
    by = g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum")
    bu = units[col[[h for h in hdr if h.startswith("dram__bytes_read.sum")][0]]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
    gbs = by * scale / (us * 1e-6) / 1e9 if us else 0
    tens = g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
    issue = g(r, "sm__inst_issued.avg.pct_of_peak_sustained_active")
    occ = g(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    st = []
    for h in hdr:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(r[col[h]]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    print(f"{name:44s} {us:7.1f} {gbs:7.0f} {100*gbs/6459.9:5.1f} {tens:5.1f} {issue:6.1f} {occ:5.1f}  " + ", ".join(f"{n}={v:.1f}" for v, n in st[:3]))
