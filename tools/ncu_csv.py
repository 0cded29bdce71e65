"""Compact per-kernel CSV of an ncu --set full report (the summary committed under profiles/)."""
import csv, io, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "sm__inst_issued.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
w = csv.writer(open(out, "w"))
M = [m for m in M if m in h]
w.writerow(["kernel"] + [f"{m} [{u[h.index(m)]}]" for m in M] + ["top_stalls"])
for r in rows[2:]:
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    w.writerow([r[h.index("Kernel Name")][:80]] + [r[h.index(m)] for m in M] + ["; ".join(f"{n}={v:.2f}" for v, n in st[:4])])
print("wrote", out)
