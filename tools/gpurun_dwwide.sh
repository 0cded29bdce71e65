# dW wide-variant check: parity with it forced on everywhere, then kernel times on c3/c4
RNNT_DW_WIDE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
RNNT_DW_PFMODE=3 timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -3
for c in ${CFGS:-3 4}; do
  for m in ${MODES:-0 1 3}; do
    echo "mode=$m c$c $(RNNT_DW_PFMODE=$m python tools/kernel_time.py $c joiner_dw_gemm)"
  done
done
