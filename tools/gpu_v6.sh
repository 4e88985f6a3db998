O=gpurun_out/v6; mkdir -p $O
python tools/cond32_probe.py > $O/cond32.json 2>&1
for f in 1 0; do SGS_RAD_FUSED=$f timeout 300 python bench.py --config c0r --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_c0r_fused$f.json 2> $O/bench_c0r_fused$f.err; done
SGS_FORCE_COMM=1 timeout 600 python bench.py --config c2 --columns 100 --steps 3 --warmup 1 --no-cpu > $O/bench_c2m100_comm1.json 2> $O/bench_c2m100_comm1.err
SGS_FORCE_COMM=1 timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu --no-e2e > $O/bench_c1_comm1.json 2> $O/bench_c1_comm1.err
SGS_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --columns 60 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/bench_c2_gloo2.json 2> $O/bench_c2_gloo2.err
timeout 900 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_comm_ordering.py tests/test_gpu_rgs.py tests/test_gpu_full_size.py -k "not c2_full and not c4_shape" -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
echo done
