import json,sys
for f in sys.argv[1:]:
    try:
        j=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    c=j.get('fusion_compare') or {}; r=j['roofline']
    print(f, 'GTEPS=%.2f ms=%.2f kms=%.2f frac=%.4f'%(j['value'], j['ms_per_step'], r['kernel_ms'], r['frac']),
      'fused', {k:c['fused'][k] for k in ('gpu_ms','buckets','rounds','grid_syncs','fused_subrounds','spills')} if c else '',
      'unfused', {k:c['unfused'][k] for k in ('gpu_ms','rounds','grid_syncs')} if c else '', 'ctas', j['counters']['ctas'])
