# r02 measurement checkpoint: gpurun_final.sh (smoke, GPU tests, c5 bench + launch list, c3/c4/dyn/full/ref
# lines), the c5 step timeline, and ncu --set full traffic for c5 and c3
bash tools/gpurun_final.sh
SKIP_FULL=1 bash tools/gpurun_r2b.sh
