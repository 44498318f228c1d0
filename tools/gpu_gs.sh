cd $GRAFT_REPO_ROOT
R=${R:-r17}
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
  timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
  for n in 256 512; do timeout 120 python tools/probe.py --n $n --depths none --gs --gs-iters 8 2>&1 | tail -2; done
) > gpurun_out/${R}_gs.log 2>&1
cat gpurun_out/${R}_gs.log
