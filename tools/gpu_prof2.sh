cd $GRAFT_REPO_ROOT
R=${R:-r15}
CMD4="python tools/probe.py --n 512 --iters 4 --depths 4 --reps 1"
CMD2="python tools/probe.py --n 512 --iters 4 --depths 2 --reps 1"
$CMD4 > gpurun_out/${R}_plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 1 -c 1 -o gpurun_out/${R}_jac4 $CMD4 > gpurun_out/${R}_ncu4.log 2>&1
$CMD2 > gpurun_out/${R}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 2 -c 1 -o gpurun_out/${R}_jac2 $CMD2 > gpurun_out/${R}_ncu2.log 2>&1
ls gpurun_out | grep $R
