for c in 2 4; do timeout 300 python tools/all_kernels.py $c; timeout 120 python tools/step_timeline.py $c; done
