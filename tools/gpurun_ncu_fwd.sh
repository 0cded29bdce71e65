ncu --set full --clock-control none --import-source on -k regex:joiner_fwd -s 2 -c 1 -o gpurun_out/fwd4_full python tools/fwd_modes.py 4 > gpurun_out/ncu_fwd4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:joiner_fwd -s 2 -c 1 -o gpurun_out/fwd2_full python tools/fwd_modes.py 2 > gpurun_out/ncu_fwd2.log 2>&1
