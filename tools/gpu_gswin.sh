cd $GRAFT_REPO_ROOT
( for w in 1000000 16 8 4 2; do echo "window=$w"; SB_GS_WINDOW=$w timeout 120 python tools/probe.py --n 512 --depths none --gs --gs-iters 100 2>&1 | tail -2; done ) > gpurun_out/${R}_gswin.log 2>&1; cat gpurun_out/${R}_gswin.log
