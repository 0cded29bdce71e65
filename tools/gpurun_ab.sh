# A/B: the current build against build_ab/librnnt_old.so on one box, kernel $1, configs $2...
k=$1; shift
for c in "$@"; do
  for rep in 1 2; do
    echo "new $(python tools/kernel_time.py $c $k)"
    echo "old $(RNNT_LIB=build_ab/librnnt_old.so python tools/kernel_time.py $c $k)"
  done
done
