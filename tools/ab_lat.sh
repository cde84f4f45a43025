L=paper_2604_27441_b200/lib
for r in 1 2; do for v in a o; do cp $L/var/lib_$v.so $L/libnvrec_b200.so; timeout 300 python bench.py --steps 100 --warmup 5 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$v',round(d['value']),round(d['value_frame_barrier']),round(d['e2e']['value']),round(d['e2e_receiver']['value']),'p50 %.3f dev %.3f'%(d['p50_latency_ms'],d['p50_latency_device_ms']))"; done; done
