# round-2 validation pass (one GPU): probes, the whole GPU suite, bench lines
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
lscpu | head -20 > $O/lscpu.txt; free -g >> $O/lscpu.txt
python tools/srht_bench.py > $O/sketch_new.json 2>&1
SGS_SRHT_LEGACY=1 SGS_DENSE_LEGACY=1 python tools/srht_bench.py > $O/sketch_legacy.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 > $O/bench_c0.json 2> $O/bench_c0.err
for f in 1 0; do SGS_RAD_FUSED=$f timeout 300 python bench.py --config c0r --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_c0r_fused$f.json 2> $O/bench_c0r_fused$f.err; done
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider -rf --durations=25 > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_c1.json 2> $O/ref_c1.err
echo done
