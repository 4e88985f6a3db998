# c3 A/B: the sketch of w on a small grid (SGS_W_SMALL_GRID=1) or one tile per CTA (0)
O=gpurun_out/${1:-c3ab}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_checked.py tests/test_gpu_krylov.py tests/test_gpu_krylov_lagged.py tests/test_gpu_sketch.py tests/test_gpu_sharded_krylov.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for v in 1 0; do
  SGS_W_SMALL_GRID=$v timeout 600 python tools/timeline_gmres_lagged.py mixed > $O/tl_lag_mixed_w$v.json 2>&1
  SGS_W_SMALL_GRID=$v timeout 600 python tools/timeline_gmres_lagged.py f64 > $O/tl_lag_f64_w$v.json 2>&1
  SGS_W_SMALL_GRID=$v timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3_w$v.json 2> $O/bench_c3_w$v.err
done
echo done
