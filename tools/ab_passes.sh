for i in 1 2; do
  for p in 32 40 24; do
    python bench.py --steps 10 --warmup 3 --no-deform --no-cpu --no-train --passes $p > gpurun_out/abp_$p$i.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/abp_$p$i.json').read().strip().splitlines()[-1]);print('$p', d['value'], d['e2e']['value'])" >> gpurun_out/abp_summary.txt
  done
done
