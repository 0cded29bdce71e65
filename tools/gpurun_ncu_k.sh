# ncu --set full of the kernels matching $KRE in one c$CFG step; compact CSV + per-kernel source hot spots
make -j16 -C paper_2206_13236_b200 > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
CFG=${CFG:-5}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KRE}" -c ${NCU_C:-8} -o gpurun_out/k_full -f python tools/one_step.py $CFG 0 > gpurun_out/ncu_k.log 2>&1; echo ncu rc $?
python tools/ncu_csv.py gpurun_out/k_full.ncu-rep gpurun_out/k_full.csv
cat gpurun_out/k_full.csv
for k in ${SRC_KERNELS:-}; do
  echo "== source hot spots: $k"; python tools/ncu_lines.py gpurun_out/k_full.ncu-rep "$k" 20 2>&1 | head -30
done
rm -f gpurun_out/k_full.ncu-rep
