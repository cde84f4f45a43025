# bash tools/sweep_env.sh VAR v1 v2 ...: bench line per value
mkdir -p gpurun_out
V=$1; shift
for x in "$@"; do echo -n "$V=$x "; env $V=$x timeout 300 python bench.py --steps 30 --warmup 5 2>>gpurun_out/ab_err.txt | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=d['stage_ms_per_step'];print(round(d['value']),round(d['ms_per_step'],4),' '.join('%s=%.4f'%(k,v) for k,v in s.items()))"; done
