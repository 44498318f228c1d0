cd $GRAFT_REPO_ROOT
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
  timeout 300 python tools/gs_shapes.py 2>&1
  timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 ) > gpurun_out/${R}_shapes.log 2>&1; cat gpurun_out/${R}_shapes.log
