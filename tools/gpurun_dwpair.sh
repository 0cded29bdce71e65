timeout 600 python -m pytest tests -m gpu -x -q -k "stagewise or edge or sampled or full_loss_small" > gpurun_out/gputest_dw.log 2>&1; echo tests=$?
for c in 2 4; do RNNT_DW_PAIR=0 timeout 300 python tools/fwd_modes.py $c joiner_dw_gemm; timeout 300 python tools/fwd_modes.py $c joiner_dw_gemm; done > gpurun_out/dw_pair.log 2>&1
