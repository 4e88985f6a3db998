# Round-2 closing pass (one GPU, final code): GPU suite, smoke, bench lines, reference arm, c1 launch list and timelines.
O=gpurun_out/final4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > $O/smi.txt 2>&1
SGS_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=15 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 > $O/bench_c0.json 2> $O/bench_c0.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --impl reference > $O/ref_default.json 2> $O/ref_default.err
python tools/timeline.py c1 > $O/tl_c1.json 2>&1
python tools/timeline_gmres_lagged.py mixed > $O/tl_gmres_lag_mixed.json 2>&1
B1="python bench.py --config c1 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2200 --csv --log-file $O/c1_launches.csv $B1 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ls_step_kernel" -s 300 -c 1 -o $O/c1_ls -f $B1 > $O/ncu_c1_ls.log 2>&1
echo done
