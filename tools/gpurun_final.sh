# end-of-round measurement: gpurun_full.sh, then the c3 / c4 / dynamic / full-loss / reference lines
bash tools/gpurun_full.sh
for c in 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.log 2>&1; echo bench c$c rc $?; done
timeout 600 python bench.py --workload dynamic --no-cpu-baseline > gpurun_out/bench_dyn.log 2>&1; echo dyn rc $?
timeout 600 python bench.py --workload full --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo full rc $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc $?
