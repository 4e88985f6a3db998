O=gpurun_out/r02l; mkdir -p $O; rm -f $O/fused2_ab.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2 > $O/pytest_fused2.txt
for rep in 1 2; do for pl in 2 1; do
  SGS_LS_PLAIN=$pl timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1 plain',$pl,round(d['value'],1))" >> $O/fused2_ab.txt
done; done
for pl in 2 1; do
  SGS_LS_PLAIN=$pl timeout 600 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 plain',$pl,{k:round(v['steps_per_s'],1) for k,v in d['results'].items()}, [v['iterations'] for v in d['results'].values()])" >> $O/fused2_ab.txt
done
echo done
