# full validation: build, smoke, all GPU tests, the default bench line, and the ncu launch list of the bench
set -x
python -c 'import __graft_entry__ as g; g.build(); g.smoke()' > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1500 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -n 3 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph --no-standalone > gpurun_out/ncu_launch.log 2>&1; echo ncu rc $?
