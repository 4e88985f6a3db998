O=gpurun_out/r02m; mkdir -p $O
timeout 100 python tools/ls_variant_probe.py > $O/probe.txt 2>&1
timeout 300 python tools/trace_ls.py c1 > $O/trace.json 2>&1
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1',round(d['value'],1))" >> $O/bench.txt
done
echo done
