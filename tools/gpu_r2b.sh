# round-2 pass b: certification-fusion tests, c1 LS timeline/trace, memcheck
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_rgs.py tests/test_gpu_certification.py tests/test_gpu_sketch.py tests/test_gpu_krylov_variants.py -q --timeout 600 -p no:cacheprovider -x > $O/pytest.log 2>&1; echo pytest_rc=$? >> $O/pytest.log
timeout 300 python tools/timeline.py c1 > $O/timeline_c1.json 2>&1
timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_c1.json 2>&1
bash tools/sanitize.sh memcheck > $O/san_memcheck.out 2>&1
cp -r gpurun_out/san $O/ 2>/dev/null
echo done
