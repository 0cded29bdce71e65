# full GPU check: smoke, all GPU tests, the default bench line and the dynamic-batch line
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo tests=$?
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --workload dynamic > gpurun_out/bench_dyn.log 2>&1; echo dyn=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
