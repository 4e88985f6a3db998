# Re-entry validation on one GPU with the current HEAD: GPU suite, smoke, bench lines.
O=gpurun_out/r02d; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/smi.txt 2>&1
SGS_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=30 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 > $O/bench_c0.json 2> $O/bench_c0.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 > $O/bench_c3.json 2> $O/bench_c3.err
python tools/timeline.py c1 > $O/tl_c1.json 2>&1
echo done
