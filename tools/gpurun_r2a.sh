set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -5 gpurun_out/gpu_tests.log
timeout 300 python tools/probe_symm.py > gpurun_out/probe_symm.log 2>&1; echo probe rc $?; cat gpurun_out/probe_symm.log | tail -3
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?; tail -c 3000 gpurun_out/bench.log
