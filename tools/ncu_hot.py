"""Top SASS instructions by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_hot.py report.ncu-rep <kernel-substring> [top=40] [context=0]"""
import csv, io, subprocess, sys

rep, key = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if row and row[0] == "Kernel Name":
        cur = [row[1], None, []]
        blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = row
    elif cur is not None:
        cur[2].append(row)
for name, hdr, rows in blocks:
    if key not in name:
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si] or 0) for r in rows)
    print("==", name[:100], "total samples", tot, "instructions", len(rows))
    idx = sorted(range(len(rows)), key=lambda i: -int(rows[i][si] or 0))[:top]
    for i in sorted(idx):
        r = rows[i]
        print(f"{i:5d} {int(r[si] or 0):6d} {100.0 * int(r[si] or 0) / max(tot, 1):5.1f}%  {r[1].strip()}")
    break
