# iteration loop: build, GPU tests, the c5 timeline (A/B variants in $TL_ENVS), per-kernel times ($CFGS)
make -j16 -C paper_2206_13236_b200 > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${TEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
  tail -n 4 gpurun_out/gpu_tests.log
fi
for e in ${TL_ENVS:-NONE=0}; do
  env $e timeout 300 python tools/timeline.py 5 > gpurun_out/timeline_c5_$e.txt 2>&1; echo "timeline $e rc $?"
  grep -v Warn gpurun_out/timeline_c5_$e.txt | grep -v warn | head -40
done
CFGS=${CFGS:-5} bash tools/kt.sh
