# Givens chain from registers: c3 standard timelines, c3 bench, GMRES GPU tests.
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_krylov_variants.py tests/test_gpu_full_size.py -k "krylov or gmres or c3 or restarted or arnoldi" -q -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python tools/timeline_gmres.py f64 > $O/tl_gmres_f64.json 2>&1
timeout 300 python tools/timeline_gmres.py mixed > $O/tl_gmres_mixed.json 2>&1
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
echo done
