# iteration: build, GPU tests, the step timeline of each config in $TL_CFGS under each env of $TL_ENVS,
# per-kernel times ($CFGS)
make -j16 -C paper_2206_13236_b200 > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
  tail -n 4 gpurun_out/gpu_tests.log
fi
for e in ${TL_ENVS:-NONE=0}; do
  for c in ${TL_CFGS:-5}; do
    env $e timeout 300 python tools/timeline.py $c > gpurun_out/timeline_c${c}_$e.txt 2>&1; echo "timeline c$c $e rc $?"
    grep -v Warn gpurun_out/timeline_c${c}_$e.txt | grep -v warn | head -40
  done
done
CFGS=${CFGS:-5} bash tools/kt.sh
