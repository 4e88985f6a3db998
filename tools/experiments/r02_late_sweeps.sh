# Late round-2 A/B sweeps on one B200 (each block ran in one gpurun call; results in
# profiles/r02i_prefetch_pacing.txt, r02k_dense_prefetch.txt, r02k_ls_rows_per_cta.txt,
# r02k_dmma_subchunks.txt, r02l_ls_plain_variant.txt).  All switches are read once per process.
B="python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e"
val() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', round(d['value'],1))"; }
# SRHT column kernel: L2 prefetch budget x pace (cycles between a tile's 16 KB prefetches)
for rep in 1 2; do for mb in 80 96 104 112 120; do for pace in 0 300 400 500; do
  SGS_COL_PF_MB=$mb SGS_COL_PF_PACE=$pace $B 2>/dev/null | val "c1 mb=$mb pace=$pace"; done; done; done
# dense ring kernel: prefetch budget
for rep in 1 2; do for mb in 0 48 80 104 128; do
  SGS_DENSE_PF_MB=$mb $B --config c0 2>/dev/null | val "c0 dense_pf_mb=$mb"; done; done
# LS cluster: rows of the k-vectors per CTA (k = 600 at c0 and c3)
for rows in 96 64 48 38; do
  SGS_LS_ROWS=$rows $B --config c0 2>/dev/null | val "c0 ls_rows=$rows"
  SGS_LS_ROWS=$rows python bench.py --config c3 --steps 3 --warmup 1 --no-cpu --no-e2e 2>/dev/null | val "c3 ls_rows=$rows"; done
# DMMA P = Theta W: sub-chunk cap
for ms in 296 152 104 72 40; do SGS_MMA_MAXSUB=$ms python tools/experiments/dmma_sub.py; done
# LS kernel variants: 2 = PLAIN + FUSED (default), 1 = PLAIN, 0 = full
for rep in 1 2 3; do for pl in 2 1 0; do SGS_LS_PLAIN=$pl $B 2>/dev/null | val "c1 ls_plain=$pl"; done; done
