import sys, json
for line in sys.stdin:
    line = line.strip()
    if line.startswith('{'):
        d = json.loads(line)
        print('value', d['value'], 'ms/step', d['ms_per_step'], 'e2e', d['e2e']['value'])
        r = d['roofline']
        print('stages(ms/step)', r.get('stage_ms_per_step'))
        print('roof', {k: r.get(k) for k in ('kernel', 'achieved', 'frac', 'avg_launch_ms')})
        if d.get('train'):
            print('train', d['train']['iters_per_s'], d['train']['stage_ms_per_iter'])
        print('detail', d['detail'], d['clocks'], d['gpu_launches'], 'cpu', d.get('cpu_baseline'))
    elif line:
        print(line)
