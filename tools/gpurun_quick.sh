# parity + c2/c4 kernel times of $KERNELS + bench c2
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for k in ${KERNELS:-prune_gather}; do for c in ${CFGS:-2 4}; do echo "$(timeout 120 python tools/kernel_time.py $c $k)"; done; done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c1-230
