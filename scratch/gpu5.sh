for cfg in "rolled-direct1::1" "rolled-direct32::32" "unrolled-direct1:scratch/libzkl_unrolled.so:1"; do
  name=${cfg%%:*}; rest=${cfg#*:}; lib=${rest%%:*}; dm=${rest#*:}
  echo "== $name"
  ZKL_LIB=$( [ -n "$lib" ] && echo $PWD/$lib ) ZKL_DIRECT_POLL_MAX=$dm timeout 300 python scratch/trace2.py 2>&1 | grep "native=True"
  ZKL_LIB=$( [ -n "$lib" ] && echo $PWD/$lib ) ZKL_DIRECT_POLL_MAX=$dm ZKL_TRACE=1 timeout 300 python scratch/trace2.py 2>&1 | grep "zkl trace" | sed -n 9,11p
done
