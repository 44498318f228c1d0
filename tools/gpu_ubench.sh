cd $GRAFT_REPO_ROOT
timeout 120 ./tools/ubench/ubench > gpurun_out/${R}_ubench.log 2>&1; cat gpurun_out/${R}_ubench.log
