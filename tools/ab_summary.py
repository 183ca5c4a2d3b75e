import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        pk=d['roofline']['per_kernel']
        print(f, round(d['value']), 'ms', round(d['ms_per_step'],3), {k:round(v['ms'],3) for k,v in pk.items()}, (d.get('parity') or {}).get('mismatched_queries'), d['gpu_launches'])
    except Exception as e:
        print(f, 'ERR', e)
