# c3 step timelines (standard f64 / mixed, lagged mixed) and the c0 e2e leg per call.
O=gpurun_out/r02e; mkdir -p $O
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 --no-cpu > $O/bench_c0.json 2> $O/bench_c0.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 --no-cpu > $O/bench_c0b.json 2> $O/bench_c0b.err
timeout 300 python tools/timeline_gmres.py f64 > $O/tl_gmres_f64.json 2>&1
timeout 300 python tools/timeline_gmres.py mixed > $O/tl_gmres_mixed.json 2>&1
timeout 300 python tools/timeline_gmres_lagged.py mixed > $O/tl_gmres_lag_mixed.json 2>&1
timeout 300 python tools/timeline_gmres_lagged.py f64 > $O/tl_gmres_lag_f64.json 2>&1
echo done
