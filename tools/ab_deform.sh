set -e
mkdir -p gpurun_out
python -m pytest tests/test_gpu_deform.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/abd_tests.log
for i in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export TSB_GEMM_WS=0; else unset TSB_GEMM_WS; fi
    echo "$v$i $(python tools/bench_deform.py 2>&1 | tail -1)" >> gpurun_out/abd_summary.txt
  done
done
