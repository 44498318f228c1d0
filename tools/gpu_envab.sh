cd $GRAFT_REPO_ROOT
# A/B of an environment toggle ($ENVAB, e.g. SB_NO_ITEMLIST=1) on the same library,
# alternating, depths $DEPTHS at sizes $NS
R=${R:-ab}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_pytest.log
tail -2 gpurun_out/${R}_pytest.log
for rep in 1 2 3; do
  for arm in new old; do
    for d in ${DEPTHS:-4}; do for n in ${NS:-1024}; do
      if [ $arm = old ]; then
        env $ENVAB timeout 300 python tools/probe.py --n $n --iters 12 --depths $d --reps 3 2>&1 | tail -1 | sed "s/^/$arm n=$n /"
      else
        timeout 300 python tools/probe.py --n $n --iters 12 --depths $d --reps 3 2>&1 | tail -1 | sed "s/^/$arm n=$n /"
      fi
    done; done
  done
done
