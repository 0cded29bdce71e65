# per-kernel standalone / live times of bench.py for the configs given in CFGS (default "5 3 4")
for c in ${CFGS:-5 3 4}; do
  timeout 400 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/kt_c$c.json 2> gpurun_out/kt_c$c.err
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
l = [x for x in open(f"gpurun_out/kt_c{c}.json") if x.startswith("{")]
if not l:
    print("c%s: no line" % c); print(open(f"gpurun_out/kt_c{c}.err").read()[-2000:]); sys.exit()
d = json.loads(l[-1])
print(f"c{c}: {d['ms_per_step']:.4f} ms/step (eager {d['eager_ms_per_step']:.4f}, serial {d['serial_ms_per_step']:.4f}), {d['value']/1e6:.2f} M frames/s")
for k, v in d["kernels"].items():
    sa = v["standalone_ms"] or 0
    print(f"   {k:22s} live {v['live_ms']*1e3:8.1f}  alone {sa*1e3:8.1f}  frac {v['frac'] if v['frac'] is None else round(v['frac'],3)}  alone_frac {v.get('standalone_frac') and round(v['standalone_frac'],3)}")
PY
done
