# A/B the bench over an environment switch: bash tools/ab_env.sh VAR valA valB [rounds]
mkdir -p gpurun_out
for r in $(seq ${4:-2}); do for v in $2 $3; do env $1=$v timeout 300 python bench.py --steps 30 --warmup 5 2>>gpurun_out/ab_err.txt | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=d['stage_ms_per_step'];print('$1=$v',round(d['value']),round(d['e2e']['value']),round(d['e2e_receiver']['value']),d['ms_per_step'],' '.join('%s=%.4f'%(k,v) for k,v in s.items()))"; done; done
