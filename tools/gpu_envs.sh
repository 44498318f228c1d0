cd $GRAFT_REPO_ROOT
# one probe line per environment setting in $ENVS (";"-separated), repeated $REPS times
IFS=';' read -ra SETS <<< "$ENVS"
for rep in $(seq ${REPS:-2}); do
  for e in "${SETS[@]}"; do
    for d in ${DEPTHS:-4}; do for n in ${NS:-1024}; do
      env $e timeout 300 python tools/probe.py --n $n --iters ${ITERS:-12} --depths $d --reps 3 2>&1 | tail -1 | sed -E 's/"hbm_frac_algo.*//' | sed "s/^/[$e] n=$n /"
    done; done
  done
done
