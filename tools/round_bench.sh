# Round bench + profiling pass (run under gpurun on one GPU):
#   gpurun --timeout 3000 -- 'bash tools/round_bench.sh gpurun_out/r01c'
set -u
O=${1:-gpurun_out/r01c}
mkdir -p $O
for c in c1 c0 c0r c2 c3; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err || echo "bench $c failed"
  tail -1 $O/bench_$c.json | cut -c1-300
done
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -1 $O/bench_ref.json | cut -c1-200
bash tools/profile_round.sh $O/prof
