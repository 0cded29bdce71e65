# bench line + launch list + one full ncu capture of every library kernel of one c2 step
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
python tools/launch_summary.py gpurun_out/launches.csv 3 > gpurun_out/launch_table.md 2>&1
ncu --set full --clock-control none --import-source on -s 40 -c 20 -o gpurun_out/step_full python tools/one_step.py 2 2 > gpurun_out/ncu_step.log 2>&1; echo ncuf=$?
