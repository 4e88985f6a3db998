# LS post-wait shortening A/B: parity tests, LS trace, c1 timeline, short benches.
O=gpurun_out/r02i; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_c1_new.json 2>&1
timeout 300 python tools/timeline.py > $O/c1_timeline_new.json 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/bench_c1_new.json 2> $O/bench_c1_new.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e > $O/bench_c3_new.json 2> $O/bench_c3_new.err
echo done
