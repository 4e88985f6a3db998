O=gpurun_out/r02j; mkdir -p $O
timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_cold.json 2>&1
SGS_LS_WARM=1 timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_warm.json 2>&1
SGS_LS_TOUCH=1 timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_touch.json 2>&1
SGS_LS_WARM=1 SGS_LS_TOUCH=1 timeout 300 python tools/trace_ls.py c1 > $O/trace_ls_both.json 2>&1
echo done
