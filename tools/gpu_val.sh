# one validation pass on the GPU box: kernel probes, the GPU test suite, the
# default bench line and the reference arm (outputs under gpurun_out/$1)
O=gpurun_out/${1:-val}
mkdir -p $O
python tools/srht_bench.py > $O/sketch_new.json 2>&1
SGS_SRHT_LEGACY=1 SGS_DENSE_LEGACY=1 python tools/srht_bench.py > $O/sketch_legacy.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 > $O/bench_c0.json 2> $O/bench_c0.err
[ -n "$REF" ] && timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_c1.json 2> $O/ref_c1.err
echo done
