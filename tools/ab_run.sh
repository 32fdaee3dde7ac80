set -e
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab_tests.log
for i in 1 2 3; do
  for v in new old; do
    if [ $v = old ]; then export TSB_LIB=$PWD/build_var/s13/libtsb.so; else unset TSB_LIB; fi
    python bench.py --steps 10 --warmup 3 --no-deform --no-cpu > gpurun_out/ab_$v$i.json 2>/dev/null
    python - <<PY >> gpurun_out/ab_summary.txt
import json;d=json.loads(open("gpurun_out/ab_$v$i.json").read().strip().splitlines()[-1]);t=d.get("train") or {}
print("$v$i", d["value"], d["e2e"]["value"], t.get("iters_per_s"), (t.get("c2") or {}).get("iters_per_s"))
PY
  done
done
