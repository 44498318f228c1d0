cd $GRAFT_REPO_ROOT
# GS probe per environment setting in $ENVS (";"-separated), ${N:-512}^3 x ${IT:-100} sweeps
IFS=';' read -ra SETS <<< "$ENVS"
for rep in $(seq ${REPS:-2}); do
  for e in "${SETS[@]}"; do
    env $e timeout 300 python tools/probe.py --n ${N:-512} --depths none --gs --gs-iters ${IT:-100} 2>&1 | grep naive | sed -E 's/"roof1_frac.*//' | sed "s/^/[$e] /"
  done
done
