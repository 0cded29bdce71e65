# every GPU test, then the bench lines of all workloads
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo tests=$?
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --workload dynamic > gpurun_out/bench_dyn.log 2>&1; echo dyn=$?
python bench.py --workload full --steps 5 > gpurun_out/bench_full.log 2>&1; echo full=$?
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
python bench.py --config 4 --no-cpu-baseline --steps 5 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
