# ncu --set full of the wide dW kernel at c4
ncu --set full --clock-control none --import-source on -k regex:joiner_dw_wide -s 3 -c 1 -o gpurun_out/dw4_full python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-graph > gpurun_out/ncu_dw4.log 2>&1; echo ncu=$?
