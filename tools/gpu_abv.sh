cd $GRAFT_REPO_ROOT
# A/B of two SB_JCFG variants, alternating, depth $D
for rep in 1 2 3; do for v in $VA $VB; do for n in ${NS:-1024 512}; do
  SB_JCFG=$v timeout 300 python tools/probe.py --n $n --iters 12 --depths $D --reps 3 2>&1 | tail -1 | sed "s/^/v$v n=$n /"
done; done; done
