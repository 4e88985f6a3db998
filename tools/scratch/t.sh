O=gpurun_out/r02k; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
echo done
