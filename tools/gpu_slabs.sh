cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_slabs.py > gpurun_out/${R}_slabs.log 2>&1; cat gpurun_out/${R}_slabs.log
