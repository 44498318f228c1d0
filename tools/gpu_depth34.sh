# sustained depth 3 vs 4: the bench headline (10 x 100 sweeps at 1024^3) and
# 512^3 (300-sweep probe runs), alternating
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for d in 3 4; do
    python bench.py --depth $d --no-cpu --no-also --no-e2e > gpurun_out/d34_bench_d${d}_r${rep}.json 2>/dev/null
    python tools/probe.py --n 512 --iters 300 --depths $d --reps 3 > gpurun_out/d34_512_d${d}_r${rep}.log 2>&1
  done
done
