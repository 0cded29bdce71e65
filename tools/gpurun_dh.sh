timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 2 3 4; do echo "$(timeout 120 python tools/kernel_time.py $c joiner_dh_gemm)"; done
timeout 120 python tools/dh_trace.py 2>&1 | sed -n 1,6p
timeout 120 python tools/dh_trace.py 2>&1 | grep -A6 "stage D4"
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-200
