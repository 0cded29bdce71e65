# pair dh: parity (hard timeouts), then kernel times and bench lines
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3 || exit 1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 2 3 4; do
  for pr in 0 1; do
    echo "pair=$pr c$c $(RNNT_DH_PAIR=$pr timeout 120 python tools/kernel_time.py $c joiner_dh_gemm)"
  done
done
for c in 2 3 4; do timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-230; done
