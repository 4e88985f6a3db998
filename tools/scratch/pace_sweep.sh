O=gpurun_out/r02i; mkdir -p $O; rm -f $O/pace_sweep3.txt
for rep in 1 2; do for mb in 96 104 112; do for pace in 200 300 400 500 600; do
  SGS_COL_PF_MB=$mb SGS_COL_PF_PACE=$pace timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mb',$mb,'pace',$pace,round(d['value'],1),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> $O/pace_sweep3.txt
done; done; done
echo done
