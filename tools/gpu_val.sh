set -x
mkdir -p gpurun_out/v2
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/v2/smi.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/dmma_probe tools/dmma_probe.cu && /tmp/dmma_probe 1500 | python tools/dmma_probe.py > gpurun_out/v2/dmma.txt 2>&1
python tools/srht_bench.py > gpurun_out/v2/srht_new.json 2>&1
SGS_SRHT_LEGACY=1 python tools/srht_bench.py > gpurun_out/v2/srht_legacy.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/v2/pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/v2/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/v2/bench_c1.json 2> gpurun_out/v2/bench_c1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/v2/ref_c1.json 2> gpurun_out/v2/ref_c1.err
echo done
