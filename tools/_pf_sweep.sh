one() { SGS_COL_PF_MB=$1 timeout 300 python bench.py --config $2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1 $2', round(d['value'],1), round(d['ms_per_step'],2), d.get('e2e',{}).get('value'))"; }
for mb in 0 32 64 96 128 0 64; do one $mb c0; done
