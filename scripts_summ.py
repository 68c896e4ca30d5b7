import json,sys
d=json.loads([l for l in open('gpurun_out/bench.log').read().strip().splitlines() if l.startswith('{')][-1])
for k in ['value','ms_per_step','stages_ms','loop_phases_us','clocks']: print(k, d.get(k))
print('e2e', d['e2e']['value'], 'roof', d['roofline']['frac'], d['roofline']['note'])
print('cpu', (d.get('cpu_baseline') or {}).get('value'))
s=d.get('secondary') or {}
print('cfg4', s.get('value'), s.get('ms_per_step'), s.get('stages_ms'), s.get('loop_phases_us'))
