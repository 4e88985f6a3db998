#!/bin/bash
# Profiling pass for profiles/ (run under gpurun on one GPU).  Every ncu command
# runs only after the same program exited 0 without ncu.
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
B="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 $B > "$OUT/bench_plain.log" 2>&1 || { echo "bench failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv \
  --log-file "$OUT/launches.csv" $B > "$OUT/ncu_launches.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"rgs_column|ls_step|srht_partials" -s 600 -c 3 -o "$OUT/c1_full" -f $B \
  > "$OUT/ncu_full.log" 2>&1
# ILU(0) at c3's 128^3: the factor and both sweeps
timeout 300 python tools/ilu_bench.py 128 quick > "$OUT/ilu_plain.log" 2>&1 || { echo "ilu failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"ilu_sweep" -c 2 -o "$OUT/ilu_sweep_full" -f \
  python tools/ilu_bench.py 128 quick > "$OUT/ncu_ilu.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"ilu_factor" -c 1 -o "$OUT/ilu_factor_full" -f \
  python tools/ilu_bench.py 128 quick >> "$OUT/ncu_ilu.log" 2>&1
# c3 launch list (one restarted solve each basis)
timeout 300 python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e > "$OUT/c3_plain.log" 2>&1 || { echo "c3 failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file "$OUT/c3_launches.csv" python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e \
  > "$OUT/ncu_c3.log" 2>&1
# c3 one-synchronisation (lagged) cycle: launch list, then the staged SpMV and
# the lagged LS launch in full
L="python tools/timeline_gmres_lagged.py mixed"
timeout 300 $L > "$OUT/c3_lagged_plain.log" 2>&1 || { echo "c3 lagged failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file "$OUT/c3_lagged_launches.csv" $L > "$OUT/ncu_c3_lagged.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"csr_spmv_staged|ls_step|srht_partials" -s 300 -c 3 -o "$OUT/c3_lagged_full" -f $L \
  >> "$OUT/ncu_c3_lagged.log" 2>&1
# device Rademacher sketch (c0r): bit generation and the packed-sign partials
timeout 300 python tools/rad_probe.py > "$OUT/rad_plain.log" 2>&1 || { echo "rad failed"; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"rademacher" -c 3 -o "$OUT/rad_full" -f python tools/rad_probe.py > "$OUT/ncu_rad.log" 2>&1
echo done
