# Fused SpMV + SRHT: its GPU tests, the GMRES tests, c3 timelines and bench (fused and SGS_SPMV_SRHT=0).
O=gpurun_out/r02g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmv_srht.py tests/test_gpu_krylov.py tests/test_gpu_krylov_lagged.py tests/test_gpu_krylov_variants.py tests/test_gpu_sharded_krylov.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python tools/timeline_gmres.py f64 > $O/tl_gmres_f64.json 2>&1
timeout 300 python tools/timeline_gmres_lagged.py mixed > $O/tl_gmres_lag_mixed.json 2>&1
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
SGS_SPMV_SRHT=0 timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3_unfused.json 2> $O/bench_c3_unfused.err
echo done
