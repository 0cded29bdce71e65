"""Write profiles/ncu_traffic.json: DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
of each library kernel in an ncu --set full report of the bench step (mean over the captured launches).

    python tools/ncu_traffic.py <report.ncu-rep> <config> [source-name]"""
import collections, csv, io, json, os, subprocess, sys

NAMES = {"joiner_dh_tc_kernel": "joiner_dh_gemm", "joiner_fwd_tc_kernel": "joiner_fwd_gemm",
         "joiner_fwd_pair_kernel": "joiner_fwd_gemm", "joiner_dw_wide_kernel": "joiner_dw_gemm",
         "joiner_dw_tc_kernel": "joiner_dw_gemm", "gemm3_kernel<rnnt::NormProb>": "simple_norm_gemm",
         "prune_kernel": "prune_gather", "combine_kernel": "lattice_combine", "simple_prep_kernel": "simple_prep",
         "gemm3_kernel<rnnt::AmProb>": "simple_am_grad_gemm", "gemm3_kernel<rnnt::LmProb>": "simple_lm_grad_gemm",
         "pruned_scan_kernel": "pruned_fb", "lattice_fb_kernel": "lattice_fb"}
rep, cfg = sys.argv[1], sys.argv[2]
srcname = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(rep)
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = collections.defaultdict(list)
for r in rows[2:]:
    name = r[h.index("Kernel Name")].replace("void ", "").replace("rnnt::", "", 1).split("(")[0]
    key = next((v for k, v in NAMES.items() if name.startswith(k)), None)
    if key is None:
        continue
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        b += float(r[i].replace(",", "")) * scale.get(u[i], 1)
    acc[key].append(b)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d.setdefault(f"c{cfg}", {})
for k, v in acc.items():
    d[f"c{cfg}"][k] = {"bytes": sum(v) / len(v), "launches": len(v), "source": f"profiles/{srcname}"}
json.dump(d, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(d[f"c{cfg}"], indent=1))
