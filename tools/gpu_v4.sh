O=gpurun_out/v4; mkdir -p $O
for v in "" "SGS_ACC_TWO=0" "SGS_SRHT_LEGACY=1" "SGS_ACC_TWO=0 SGS_SRHT_LEGACY=1" "SGS_LS_DEFER=0"; do env $v python tools/cond32_probe.py >> $O/cond32.jsonl 2>&1; done
timeout 1200 python -m pytest tests/test_gpu_ls.py tests/test_gpu_acceptance.py tests/test_gpu_rgs.py tests/test_gpu_sketch.py tests/test_gpu_sharded.py tests/test_gpu_edge_cases.py tests/test_gpu_certification.py "tests/test_gpu_full_size.py::test_c0_shape_device_rademacher_factorization" -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python bench.py --config c0r --steps 10 --warmup 3 --no-cpu > $O/bench_c0r.json 2> $O/bench_c0r.err
echo done
