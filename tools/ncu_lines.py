"""Aggregate ncu source-page stall samples by CUDA source line: python tools/ncu_lines.py src.csv [kernel-substring] [top]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cur_file = None; cur_fn = ""; hdr = None
agg = collections.Counter(); src = {}; execs = collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        cur_fn = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or not r[0].isdigit() or want not in cur_fn:
        continue
    try:
        samp = float(r[4] or 0)
    except ValueError:
        samp = 0
    key = (cur_file, int(r[0])); agg[key] += samp; src[key] = r[1][:90]
    try:
        execs[key] += float(r[7] or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
for k, v in agg.most_common(top):
    print(f"{v / tot:6.1%} {int(execs[k]):9d} {k[0]}:{k[1]} {src[k]}")
