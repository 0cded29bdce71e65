# A/B of one environment switch: GPU tests with the default, then c5 / c3 bench lines with the switch on and off
# usage: SW=RNNT_FWD_ARES bash tools/gpurun_ab.sh   (CFGS="5 3", TESTS=1)
SW=${SW:-RNNT_FWD_ARES}
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1; echo build rc $?
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
  tail -n 3 gpurun_out/gpu_tests.log
fi
for c in ${CFGS:-5 3}; do
  for v in ${VALS:-1 0}; do
    env $SW=$v timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ab_c${c}_$v.log 2>&1; echo c$c $SW=$v rc $?
    python - gpurun_out/ab_c${c}_$v.log <<'PY'
import json, os, sys
l = [x for x in open(sys.argv[1]).read().splitlines() if x.startswith("{")]
if l:
    d = json.loads(l[-1]); k = d["kernels"]
    print("  ms/step %.4f" % d["ms_per_step"], " ".join("%s %.1f/%.1f" % (n.replace("_gemm", ""), k[n]["live_ms"] * 1e3, k[n]["standalone_ms"] * 1e3) for n in os.environ.get("KERNELS", "joiner_fwd_gemm joiner_dh_gemm joiner_dw_gemm").split()))
PY
  done
done
