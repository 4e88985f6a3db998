O=gpurun_out/final3; mkdir -p $O
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 > $O/bench_c0_b.json 2> $O/bench_c0_b.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 --no-cpu > $O/bench_c0_c.json 2> $O/bench_c0_c.err
echo done
