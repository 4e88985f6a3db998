# Round-2 closing bench lines after the LS launch-mode variants (one GPU, final code; the GPU suite ran green on this code in the A/B call before).
O=gpurun_out/final5; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --config c0 --steps 10 --warmup 3 > $O/bench_c0.json 2> $O/bench_c0.err
timeout 900 python bench.py --config c3 --steps 3 --warmup 1 > $O/bench_c3.json 2> $O/bench_c3.err
python tools/timeline_gmres.py f64 > $O/tl_gmres_f64.json 2>&1
echo done
