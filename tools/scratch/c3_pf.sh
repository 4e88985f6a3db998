O=gpurun_out/r02j; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_krylov_lagged.py tests/test_gpu_rgs.py tests/test_gpu_spmv_srht.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3_pf.json 2> $O/bench_c3_pf.err
SGS_COL_PF_PACE=0 timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3_nopf.json 2> $O/bench_c3_nopf.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > $O/bench_c1.json 2> $O/bench_c1.err
echo done
