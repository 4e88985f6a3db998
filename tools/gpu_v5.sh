O=gpurun_out/v5; mkdir -p $O
python tools/f32_diverge.py f32 > $O/diverge_f32.json 2>&1
python tools/trace_ls.py c1 > $O/trace_ls_c1.json 2>&1
python tools/timeline.py c1 > $O/timeline_c1.json 2>&1
timeout 300 python bench.py --config c0r --steps 10 --warmup 3 --no-cpu > $O/bench_c0r.json 2> $O/bench_c0r.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err
echo done
