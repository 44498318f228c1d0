cd $GRAFT_REPO_ROOT
( timeout 120 python tools/diag_jacobi.py 40x36x30
  timeout 120 python tools/diag_jacobi.py 64x64x64
  for n in 128 256 512; do echo "probe n=$n"; timeout 60 python tools/probe.py --n $n --iters 8 --depths 1,2,4,8 --reps 2 2>&1 | tail -4; done
  timeout 120 python tools/probe.py --n 256 --depths "" --gs --gs-iters 4 2>&1 | tail -3
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
) > gpurun_out/r7_diag.log 2>&1
cat gpurun_out/r7_diag.log
