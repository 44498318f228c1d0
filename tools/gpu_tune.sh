cd $GRAFT_REPO_ROOT
R=${R:-r14}
( timeout 120 python tools/diag_jacobi.py 40x36x30
  timeout 120 python tools/diag_jacobi.py 130x70x50 0.5
  timeout 120 python tools/diag_jacobi.py 200x160x70
  for v in 0 1; do for a0 in ""; do echo "SB_JCFG=$v SB_NO_A0=$a0"; env ${a0:+SB_NO_A0=1} SB_JCFG=$v timeout 120 python tools/probe.py --n 512 --iters 8 --depths 1,2,3,4,8 --reps 3 2>&1 | tail -5; done; done
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
) > gpurun_out/${R}_tune.log 2>&1
cat gpurun_out/${R}_tune.log
