cd $GRAFT_REPO_ROOT
# k-block length sweep (SB_KBLK bypasses the picker and the item list)
for kb in ${KBS:-128 205 256 342 512 658 1024}; do
  for d in ${DEPTHS:-4}; do for n in ${NS:-1024}; do
    SB_KBLK=$kb timeout 300 python tools/probe.py --n $n --iters 12 --depths $d --reps 3 2>&1 | tail -1 | sed "s/^/kb=$kb n=$n /"
  done; done
done
for d in ${DEPTHS:-4}; do for n in ${NS:-1024}; do
  timeout 300 python tools/probe.py --n $n --iters 12 --depths $d --reps 3 2>&1 | tail -1 | sed "s/^/list n=$n /"
  SB_NO_ITEMLIST=1 timeout 300 python tools/probe.py --n $n --iters 12 --depths $d --reps 3 2>&1 | tail -1 | sed "s/^/pick n=$n /"
done; done
