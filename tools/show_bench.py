import json,sys
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith('{'):
            d=json.loads(l)
            r = d.get('roofline') or {}
            print(f.split('/')[-1], round(d['value'],1), 'it/s', round(d['ms_per_step'],3), 'ms', 'dom', r.get('kernel'), round(r.get('frac',0),3), 'step GB/s', round(d['step_algorithmic_gbs'] or 0))
            print('   ', {k:(round(v['ms_per_launch'],4), v['launches']) for k,v in d['kernels'].items()})
