import json, sys
d = json.loads(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench.log').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value', 'ms_per_step', 'dtype', 'n_gpus', 'scaling', 'gpu_launches', 'clocks')})
r = d['roofline']
print(' top:', r['kernel'][:50], 'frac=%.3f' % r['frac'], 'ms=%.4f' % r['avg_launch_ms'], 'share=%.3f' % r['share_of_step'], 'design_B', r.get('bytes_moved_by_design'))
for o in r.get('other_kernels', []):
    print('   ', o['kernel'][:50], 'frac=%.3f' % o['frac'], 'ms=%.4f' % o['avg_launch_ms'], 'share=%.3f' % o['share_of_step'])
if d.get('e2e'): print(' e2e', d['e2e']['value'])
if d.get('cpu_baseline'): print(' cpu', d['cpu_baseline']['value'], d['cpu_baseline'].get('cpu_model'))
for k, v in (d.get('configs') or {}).items():
    r = v['roofline']
    print(k, '%.3e' % v['value'], 'ms/step=%.3f' % v['ms_per_step'], v['path'][:22], '|', r['kernel'][:28], 'frac=%.3f' % r['frac'], 'share=%.2f' % r['share_of_step'], 'cpu', (v['cpu_baseline'] or {}).get('value'))
