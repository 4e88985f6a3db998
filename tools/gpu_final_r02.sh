# Round-2 evidence pass (one GPU): full GPU suite with the parity log, the
# bench lines of every config, the reference arm, a c1 launch list.
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/smi.txt 2>&1
lscpu | head -20 > $O/lscpu.txt
SGS_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=30 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 > $O/bench_c0.json 2> $O/bench_c0.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config c0r --steps 10 --warmup 3 --no-cpu > $O/bench_c0r.json 2> $O/bench_c0r.err
python tools/srht_bench.py > $O/sketch.json 2>&1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_c1.json 2> $O/ref_c1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2200 --csv --log-file $O/c1_launches.csv python bench.py --config c1 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph > $O/ncu_launch.log 2>&1
echo done
