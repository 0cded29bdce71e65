# round-1 profile refresh: GPU tests, bench lines of every workload, c2 launch list, full ncu step captures (c2, c4 joiners)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo tests=$?
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --workload dynamic > gpurun_out/bench_dyn.log 2>&1; echo dyn=$?
python bench.py --workload full --steps 5 > gpurun_out/bench_full.log 2>&1; echo full=$?
python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
python bench.py --config 4 --no-cpu-baseline --steps 5 > gpurun_out/bench_c4.log 2>&1; echo c4=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
python tools/launch_summary.py gpurun_out/launches.csv 3 > gpurun_out/launch_table.md 2>&1
ncu --set full --clock-control none --import-source on -s 40 -c 20 -o gpurun_out/step_full python tools/one_step.py 2 2 > gpurun_out/ncu_step.log 2>&1; echo ncuf=$?
ncu --set full --clock-control none --import-source on -k regex:joiner -s 6 -c 3 -o gpurun_out/c4_joiners python tools/one_step.py 4 2 > gpurun_out/ncu_c4.log 2>&1; echo ncu4=$?
