# quick GPU check: parity tests, then the bench (no e2e / cpu legs) and a launch list
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests=$?
python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
python tools/launch_summary.py gpurun_out/launches.csv 3 > gpurun_out/launch_table.md 2>&1
