# r02 validation + traffic: gpurun_full.sh, the step timeline, then ncu --set full captures of one c5 and one
# c3 step (reports deleted after their summaries are written: gpurun_out/ must stay < 64 MiB)
[ "${SKIP_FULL:-0}" = 1 ] || bash tools/gpurun_full.sh
timeout 300 python tools/timeline.py 5 > gpurun_out/timeline_c5.txt 2>&1; echo timeline rc $?
for c in ${NCU_CFGS:-5 3}; do
  timeout 900 ncu --set full --clock-control none --import-source on -c 40 -o gpurun_out/c${c}_step_full -f python tools/one_step.py $c 0 > gpurun_out/ncu_full_c$c.log 2>&1; echo ncu full c$c rc $?
  python tools/ncu_traffic.py gpurun_out/c${c}_step_full.ncu-rep $c r02_c${c}_step_ncu_full.csv > /dev/null; echo traffic c$c rc $?
  python tools/ncu_csv.py gpurun_out/c${c}_step_full.ncu-rep gpurun_out/r02_c${c}_step_ncu_full.csv
  rm -f gpurun_out/c${c}_step_full.ncu-rep
done
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
du -sh gpurun_out; ls -la gpurun_out
