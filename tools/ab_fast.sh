# A/B the fast-precision bench over prebuilt library variants: bash tools/ab_fast.sh a b [rounds]
L=paper_2604_27441_b200/lib
R=${3:-2}; mkdir -p gpurun_out
for r in $(seq $R); do for v in $1 $2; do cp $L/var/lib_$v.so $L/libnvrec_b200.so; timeout 200 python bench.py --precision fast --no-extra --steps 30 --warmup 5 2>>gpurun_out/ab_err.txt | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);s=d['stage_ms_per_step'];print('$v',round(d['value']),' '.join('%s=%.4f'%(k,v) for k,v in s.items()))"; done; done
