# ncu --set full of one kernel (regex $1) from the c2 bench step
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-3} -c ${3:-1} -o gpurun_out/one_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_one.log 2>&1; echo ncu=$?
