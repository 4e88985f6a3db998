O=gpurun_out/r02j; mkdir -p $O; rm -f $O/hint_ab.txt
for rep in 1 2; do for h in 0 1; do
  SGS_COL_PF_HINT=$h timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('hint',$h,round(d['value'],1),d['clocks']['sm_mhz'],d['clocks']['reasons'])" >> $O/hint_ab.txt
done; done
SGS_COL_PF_HINT=1 timeout 300 python tools/timeline.py > $O/c1_timeline_hint.json 2>&1
SGS_COL_PF_HINT=1 timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_hint.json 2>&1
echo done
