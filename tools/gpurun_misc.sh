timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k grad_hook 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:joiner -s 6 -c 3 -o gpurun_out/c4_joiners python tools/one_step.py 4 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu4=$?
