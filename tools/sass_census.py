"""Per-kernel SASS instruction census of the built library (cuobjdump -sass): the instructions that
prove the tensor-core / TMA / TMEM path (UTCHMMA = tcgen05.mma kind::f16, .2CTA = cta_group::2,
UTMALDG / UTMASTG = TMA tensor loads / stores, UBLKCP = bulk copies, LDTM = tcgen05.ld, UTCBAR =
tcgen05.commit) plus the exchange reductions (REDG).  Writes a markdown table to stdout.

    python tools/sass_census.py [path/to/librnnt_b200.so] > profiles/r02_sass_census.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2206_13236_b200", "librnnt_b200.so")
KEYS = ["UTCHMMA", "UTCHMMA.2CTA", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "UTCBAR",
        "REDG", "SYNCS", "MUFU", "DSETP/DFMA/DADD"]


def classify(op):
    if op.startswith("UTCHMMA"):
        return ["UTCHMMA.2CTA"] if ".2CTA" in op else ["UTCHMMA"]
    if op.startswith("UTMALDG"):
        return ["UTMALDG"]
    if op.startswith("UTMASTG"):
        return ["UTMASTG"]
    if op.startswith("UTMACCTL.PF") or op.startswith("UTMAPF"):
        return ["UTMAPF"]
    if op.startswith("UBLKCP"):
        return ["UBLKCP"]
    if op.startswith("LDTM"):
        return ["LDTM"]
    if op.startswith("STTM"):
        return ["STTM"]
    if op.startswith("UTCBAR"):
        return ["UTCBAR"]
    if op.startswith("REDG"):
        return ["REDG"]
    if op.startswith("SYNCS"):
        return ["SYNCS"]
    if op.startswith("MUFU"):
        return ["MUFU"]
    if op.startswith(("DSETP", "DFMA", "DADD", "DMUL")):
        return ["DSETP/DFMA/DADD"]
    return []


def main():
    txt = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts.setdefault(cur, collections.Counter())
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m and cur:
            for k in classify(m.group(2)):
                counts[cur][k] += 1
    dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS census of `{os.path.relpath(SO, ROOT)}` (cuobjdump -sass, sm_100a)\n")
    print("Static instruction counts per kernel (not dynamic).  UTCHMMA = tcgen05.mma (kind::f16), "
          "UTCHMMA.2CTA = cta_group::2, UTMALDG/UTMASTG = TMA tensor load/store, UTMAPF = TMA L2 prefetch, "
          "UBLKCP = cp.async.bulk, LDTM = tcgen05.ld, UTCBAR = tcgen05.commit, REDG = global reductions "
          "(the exchange's red.add / multimem.red.add, the latter on an NVLS multicast address), "
          "SYNCS = mbarrier ops.\n")
    print("| kernel | " + " | ".join(KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for (k, c), name in zip(counts.items(), dem):
        if not any(c.values()):
            continue
        short = re.sub(r"\(.*", "", name).replace("rnnt::", "")
        print(f"| `{short}` | " + " | ".join(str(c.get(x, 0)) for x in KEYS) + " |")


if __name__ == "__main__":
    main()
