# Re-entry validation at HEAD: full GPU suite, smoke, default bench, reference arm.
O=gpurun_out/r02h; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python tools/timeline.py > $O/c1_timeline.json 2>&1
echo done
