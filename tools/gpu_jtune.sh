cd $GRAFT_REPO_ROOT
( for v in ${VARIANTS:-0}; do
  echo "SB_JCFG=$v"
  SB_JCFG=$v timeout 120 python tools/diag_jacobi.py 40x36x30 | grep -v " ok$"
  SB_JCFG=$v timeout 120 python tools/diag_jacobi.py 130x70x50 0.5 | grep -v " ok$"
  SB_JCFG=$v timeout 120 python tools/diag_jacobi.py 200x160x70 | grep -v " ok$"
  SB_JCFG=$v timeout 300 python tools/probe.py --n 1024 --iters 12 --depths ${DEPTHS:-1,2,3,4} --reps 2 2>&1 | tail -4; SB_JCFG=$v timeout 300 python tools/probe.py --n 512 --iters 12 --depths ${DEPTHS:-1,2,3,4} --reps 2 2>&1 | tail -4; done
  [ -n "$PYTEST" ] && timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
) > gpurun_out/${R}_jtune.log 2>&1; cat gpurun_out/${R}_jtune.log
