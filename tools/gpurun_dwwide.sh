# dW wide-variant check: parity with it forced on everywhere, then kernel + step A/B on c2-c4
set -x
RNNT_DW_WIDE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 2 3 4; do
  for w in 0 1; do
    echo "wide=$w c$c $(RNNT_DW_WIDE=$w python tools/kernel_time.py $c joiner_dw_gemm)"
  done
done
for c in 3 4; do
  for w in 0 1; do
    echo "wide=$w c$c $(RNNT_DW_WIDE=$w python tools/step_timeline.py $c 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
for w in 0 1; do RNNT_DW_WIDE=$w python bench.py --config 4 --steps 10 --warmup 3 2>/dev/null | cut -c1-200; done
