#!/bin/bash
# Round-2 profiling pass for profiles/ (one GPU, under gpurun).  Every ncu
# command runs only after the same program exited 0 without ncu.
set -u
OUT=${1:-gpurun_out/prof2}
mkdir -p "$OUT"
B1="python bench.py --config c1 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph"
B0="python bench.py --config c0 --steps 1 --warmup 1 --no-cpu --no-e2e --no-graph"
B3="python bench.py --config c3 --steps 1 --warmup 0 --no-cpu --no-e2e"
timeout 300 $B1 > "$OUT/c1_plain.log" 2>&1 || { echo "c1 failed"; exit 1; }
# every launch of the c1 run with its device time (shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2200 --csv \
  --log-file "$OUT/c1_launches.csv" $B1 > "$OUT/ncu_c1_launches.log" 2>&1
# column 300 of the first factorisation, the LS launch after it, the P batch
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"rgs_column_kernel" -s 300 -c 1 -o "$OUT/c1_column" -f $B1 > "$OUT/ncu_c1_col.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"ls_step_kernel" -s 300 -c 1 -o "$OUT/c1_ls" -f $B1 > "$OUT/ncu_c1_ls.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"srht_tile_kernel" -c 1 -o "$OUT/c1_pbatch" -f $B1 > "$OUT/ncu_c1_pb.log" 2>&1
timeout 300 $B0 > "$OUT/c0_plain.log" 2>&1 || { echo "c0 failed"; exit 1; }
# c0: the dense ring column kernel at column 200 and the DMMA P = Theta W
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"dense_ring_kernel" -s 200 -c 1 -o "$OUT/c0_column" -f $B0 > "$OUT/ncu_c0_col.log" 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"dense_mma_kernel" -c 1 -o "$OUT/c0_dmma" -f $B0 > "$OUT/ncu_c0_dmma.log" 2>&1
timeout 600 $B3 > "$OUT/c3_plain.log" 2>&1 || { echo "c3 failed"; exit 1; }
# c3 (fp64 basis, standard RGS-Arnoldi): column 250 of the first cycle
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"rgs_column_kernel" -s 250 -c 1 -o "$OUT/c3_column" -f $B3 > "$OUT/ncu_c3_col.log" 2>&1
echo done
