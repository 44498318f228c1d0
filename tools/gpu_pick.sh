cd $GRAFT_REPO_ROOT
( for v in 0 1 2; do echo "SB_JCFG=$v"; SB_JCFG=$v timeout 300 python tools/probe.py --n 1024 --iters 12 --depths 1,2,3,4 --reps 2 2>&1 | tail -4; done
  timeout 300 python tools/probe.py --n 512 --depths none --gs --gs-iters 100 2>&1 | tail -2
  timeout 900 python -m pytest tests/test_slabs.py -x -q 2>&1 | tail -2
) > gpurun_out/${R}_pick.log 2>&1; cat gpurun_out/${R}_pick.log
