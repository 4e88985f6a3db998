# c1 column-kernel L2 prefetch budget sweep (SGS_COL_PF_MB), resident graph value
for rep in 1 2; do for mb in 64 80 96 112 128; do
  SGS_COL_PF_MB=$mb timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pf_mb', $mb, 'rep', $rep, round(d['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
