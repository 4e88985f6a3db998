O=gpurun_out/r02k; mkdir -p $O
timeout 200 python tools/scratch/dmma_sub.py > $O/dmma_stage32x2.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_sketch.py -q -p no:cacheprovider -x 2>&1 | tail -2 >> $O/dmma_stage32x2.txt
echo done
