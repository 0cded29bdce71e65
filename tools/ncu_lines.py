"""Warp-stall samples per CUDA source line of one kernel in an ncu report (--import-source on):
python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, f, tot = [], None, 0
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    stalls = sorted(((int(v) if v.isdigit() else 0, k[6:]) for k, v in zip(hdr, r) if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:3]
    rows.append((s, f, r[0], r[1].strip()[:90], stalls))
    tot += s
rows.sort(reverse=True)
print("total samples", tot)
for s, f, ln, src, st in rows[:top]:
    print(f"{s:6d} {100*s/max(tot,1):5.1f}% {f}:{ln:5s} {src}   [{', '.join(f'{k}={v}' for v, k in st if v)}]")
