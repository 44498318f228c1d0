cd $GRAFT_REPO_ROOT
for v in 0 5 6 7; do for n in 1024 512; do SB_JCFG=$v timeout 300 python tools/probe.py --n $n --iters 12 --depths 1,2 --reps 3 2>&1 | tail -2 | sed "s/^/v$v n=$n /"; done; done
