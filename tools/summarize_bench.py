import json, sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][0]
d=json.loads(l)
print('value %.3g ms/step %.2f e2e %.3g (%.2f ms)'%(d['value'],d['ms_per_step'],d['e2e']['value'] if d.get('e2e') else 0, d['e2e']['ms_per_step'] if d.get('e2e') else 0))
r=d['roofline']; print('roof frac %.3f serial_frac %.3f achieved %.2f peak %.2f'%(r['frac'],r.get('serial_frac',0),r['achieved'],r['peak']))
for name in ['kernels','kernels_serial']:
    print(name, ' total %.2f'%sum(v['ms'] for v in d[name].values()))
    for k,v in d[name].items(): print('   %-28s %7.3f ms  %s'%(k,v['ms'], '%.0f GB/s'%v['hbm_gbs'] if v['hbm_gbs'] else ''))
print(d['clocks'], d['gpu_launches'])
