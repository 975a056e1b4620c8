import json, sys
for c in (sys.argv[1:] or ['C1','C2','C3','C4','C5']):
    try: d=json.load(open(f'/root/repo/gpurun_out/bench_{c}.json'))
    except Exception as e: print(c, 'missing'); continue
    r=d['roofline']
    print(c, d['config']['iterations'], round(d['ms_per_step'],2), '%.3g'%d['value'], 'symv frac', round(r['frac'],3), 'iter GB/s', round(r['iteration_model_GBps']), {k:round(v,2) for k,v in d['kernel_ms_per_solve'].items()}, 'setup', d['config']['t_setup_s'], 'launches', d['gpu_launches'])
