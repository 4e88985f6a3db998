O=gpurun_out/r02k; mkdir -p $O; rm -f $O/dense_pf.txt
for rep in 1 2; do for mb in 0 48 80 104 128; do
  SGS_DENSE_PF_MB=$mb timeout 300 python bench.py --config c0 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c0 mb',$mb,round(d['value'],1),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> $O/dense_pf.txt
done; done
for mb in 0 48 104; do
  SGS_DENSE_PF_MB=$mb timeout 300 python bench.py --config c0r --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c0r mb',$mb,round(d['value'],1),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> $O/dense_pf.txt
done
echo done
