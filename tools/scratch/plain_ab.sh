O=gpurun_out/r02l; mkdir -p $O; rm -f $O/plain_ab.txt
timeout 900 python -m pytest tests/test_gpu_ls.py tests/test_gpu_rgs.py tests/test_gpu_sharded.py tests/test_gpu_comm_ordering.py -q -p no:cacheprovider -x 2>&1 | tail -2 > $O/pytest_plain.txt
for rep in 1 2 3; do for pl in 1 0; do
  SGS_LS_PLAIN=$pl timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1 plain',$pl,round(d['value'],1))" >> $O/plain_ab.txt
done; done
for pl in 1 0; do
  SGS_LS_PLAIN=$pl timeout 300 python bench.py --config c0 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c0 plain',$pl,round(d['value'],1))" >> $O/plain_ab.txt
done
SGS_LS_PLAIN=1 timeout 300 python tools/trace_ls.py c1 > $O/trace_plain1.json 2>&1
SGS_LS_PLAIN=0 timeout 300 python tools/trace_ls.py c1 > $O/trace_plain0.json 2>&1
echo done
