# wide dW: L2 prefetch distance / policy / grid order sweep
RNNT_DW_PFMODE=3 timeout 300 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "c4 or c3" 2>&1 | tail -2
for c in 4 3; do
  for m in 0 1 2 3; do
    for pf in 0 3 6 12; do
      echo "c$c mode=$m pf=$pf $(RNNT_DW_PFMODE=$m RNNT_DW_PF=$pf python tools/kernel_time.py $c joiner_dw_gemm)"
    done
  done
done
