cd $GRAFT_REPO_ROOT
echo "single, cluster-2 launch"; SB_FORCE_CLUSTER=1 timeout 300 python tools/probe.py --n 1024 --iters 12 --depths 1,3,4 --reps 2 2>&1 | tail -3
echo "single"; timeout 300 python tools/probe.py --n 1024 --iters 12 --depths 1,3,4 --reps 2 2>&1 | tail -3
