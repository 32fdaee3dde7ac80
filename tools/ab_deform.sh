set -e
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_deform.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/abd_tests.log
for i in 1 2; do
  for v in new old; do
    unset TSB_LIB
    if [ $v = old ]; then export TSB_LIB=$PWD/build_var/d3/libtsb.so; fi
    echo "$v$i $(timeout 120 python tools/bench_deform.py 2>&1 | tail -1)" >> gpurun_out/abd_summary.txt
  done
done
