cd $GRAFT_REPO_ROOT
for rep in 1 2; do
timeout 300 python tools/probe.py --n 1024 --iters 12 --depths 3 --reps 3 2>&1 | tail -1 | sed "s/^/auto-alone /"
SB_KBLK=395 timeout 300 python tools/probe.py --n 1024 --iters 12 --depths 3 --reps 3 2>&1 | tail -1 | sed "s/^/kb395 /"
timeout 300 python tools/probe.py --n 1024 --iters 12 --depths 2,3 --reps 3 2>&1 | tail -1 | sed "s/^/auto-after-T2 /"
done
