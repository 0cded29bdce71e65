set -x
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/fullsize.log 2>&1; echo full=$?
ncu --set full --clock-control none --import-source on -k regex:joiner_ -s 6 -c 3 -o gpurun_out/joiner_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncuf=$?
ncu --set full --clock-control none --import-source on -k regex:"pruned_fb|gemm3|combine_kernel|prune_kernel|lattice_fb|simple_prep" -s 12 -c 8 -o gpurun_out/misc_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_m.log 2>&1; echo ncum=$?
