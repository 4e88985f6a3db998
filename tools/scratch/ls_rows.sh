O=gpurun_out/r02k; mkdir -p $O; rm -f $O/ls_rows.txt
for rows in 96 64 48 38; do
  SGS_LS_ROWS=$rows timeout 600 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 rows',$rows,{k:round(v['steps_per_s'],1) for k,v in d['results'].items()}, [v['iterations'] for v in d['results'].values()])" >> $O/ls_rows.txt
  SGS_LS_ROWS=$rows timeout 300 python bench.py --config c0 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c0 rows',$rows,round(d['value'],1))" >> $O/ls_rows.txt
done
echo done
