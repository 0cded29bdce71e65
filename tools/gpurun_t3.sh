# 3-D TMA boxes in dh (W) and dW: parity, then kernel times and bench lines
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
RNNT_DW_WIDE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for c in 2 3 4; do
  echo "c$c $(python tools/kernel_time.py $c joiner_dh_gemm)"
  echo "c$c $(python tools/kernel_time.py $c joiner_dw_gemm)"
done
echo "c2 wide $(RNNT_DW_WIDE=1 python tools/kernel_time.py 2 joiner_dw_gemm)"
for c in 2 3 4; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); print(d['config']['workload'], d['ms_per_step'], d['value'], d['e2e']['value'] if d.get('e2e') else None)"; done
