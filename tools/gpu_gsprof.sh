cd $GRAFT_REPO_ROOT
timeout 300 python tools/gsprof/run.py > gpurun_out/${R}_gsprof.log 2>&1; cat gpurun_out/${R}_gsprof.log
