# LS kernel iteration: parity-critical tests, c1 timeline + phase trace, c1 bench line
O=gpurun_out/${1:-ls}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_rgs.py tests/test_gpu_ls.py tests/test_gpu_full_size.py tests/test_gpu_krylov_lagged.py tests/test_gpu_comm_ordering.py -q --timeout 600 -p no:cacheprovider -x -k "not c2_full and not c4_shape" > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 300 python tools/timeline.py c1 > $O/timeline_c1.json 2>&1
timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_c1.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_c1.json 2> $O/bench_c1.err
echo done
