set -e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab_tests.log
for i in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export TSB_BENCH_SPLIT_DL=1; else unset TSB_BENCH_SPLIT_DL; fi
    python bench.py --steps 10 --warmup 3 --no-deform --no-cpu --no-train > gpurun_out/ab_$v$i.json 2>/dev/null
    python - <<PY >> gpurun_out/ab_summary.txt
import json;d=json.loads(open("gpurun_out/ab_$v$i.json").read().strip().splitlines()[-1])
print("$v$i", d["value"], d["e2e"]["value"])
PY
  done
done
