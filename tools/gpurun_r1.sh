set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests=$?
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --profile-kernel joiner_dh_gemm --no-e2e --no-cpu-baseline > gpurun_out/bench_dh.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
ncu --set full --clock-control none --import-source on -k regex:joiner_ -s 30 -c 3 -o gpurun_out/joiner_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncuf=$?
