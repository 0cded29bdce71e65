# compute-sanitizer over one step of every path (c1 and a 4-utterance c2 shard); logs in gpurun_out/
set -x
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 python tools/sanitize_step.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc $?"
  tail -n 4 gpurun_out/sanitize_$tool.log
done
