# validation of the 4-tile SRHT groups: full GPU suite, c1/c3/c2 bench lines, sketches, c1 timeline
O=gpurun_out/${1:-tg4}; mkdir -p $O
SGS_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > $O/bench_c1.json 2> $O/bench_c1.err
timeout 300 python tools/timeline.py c1 > $O/tl_c1.json 2>&1
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python tools/timeline_gmres_lagged.py mixed > $O/tl_c3_lag_mixed.json 2>&1
timeout 900 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
python tools/srht_bench.py > $O/sketch.json 2>&1
echo done
