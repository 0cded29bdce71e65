# A/B of several kernels: the current build against build_ab/librnnt_old.so, configs $CFGS
for c in ${CFGS:-2 4}; do
  for k in $KERNELS; do
    for rep in 1 2; do
      echo "new $(python tools/kernel_time.py $c $k)"
      echo "old $(RNNT_LIB=build_ab/librnnt_old.so python tools/kernel_time.py $c $k)"
    done
  done
done
