cd $GRAFT_REPO_ROOT
for dc in 0,0,0 2,0,0 -1,0,0 0,-1,0 0,0,-1 -2,0,0 -16,0,0 500,0,0 0,0,600; do
  echo "== SB_DC=$dc"; SB_DEBUG=1024 SB_DC=$dc timeout 60 python tools/bisect_jacobi.py 1 512 2>&1 | tail -1
done > gpurun_out/r4_bisect.log 2>&1
cat gpurun_out/r4_bisect.log
