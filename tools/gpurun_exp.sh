# quick experiment runner: build, then the commands given in EXP (one per line)
set -x
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
eval "$EXP"
