cd $GRAFT_REPO_ROOT
# A/B: in-tree library vs exp/$OLD, alternating, depths $DEPTHS at n=$N
for rep in 1 2 3; do
  for lib in new old; do
    if [ $lib = old ]; then export SB200_LIB=exp/${OLD:-libsb200_old.so}; else unset SB200_LIB; fi
    for d in ${DEPTHS:-4}; do for n in ${NS:-1024}; do
      timeout 300 python tools/probe.py --n $n --iters 12 --depths $d --reps 3 2>&1 | tail -1 | sed "s/^/$lib n=$n /"
    done; done
  done
done
