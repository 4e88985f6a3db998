# LS kernel A/B on one box: parity subset, then timeline/trace/bench per variant
O=gpurun_out/${1:-lsab}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_rgs.py tests/test_gpu_ls.py tests/test_gpu_krylov_lagged.py -q --timeout 600 -p no:cacheprovider -x > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
for v in ${VARIANTS:-1 0}; do
  SGS_LS_ONEPASS=$v timeout 300 python tools/timeline.py c1 > $O/timeline_c1_op$v.json 2>&1
  SGS_LS_ONEPASS=$v timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_c1_op$v.json 2>&1
  SGS_LS_ONEPASS=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench_c1_op$v.json 2> $O/bench_c1_op$v.err
done
for v in ${VARIANTS:-1 0}; do
  SGS_LS_ONEPASS=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/bench2_c1_op$v.json 2> $O/bench2_c1_op$v.err
done
echo done
