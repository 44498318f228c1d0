cd $GRAFT_REPO_ROOT
R=${R:-r19}
CMD="python tools/probe.py --n 512 --depths none --gs --gs-iters 16"
$CMD > gpurun_out/${R}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gs_tile -s 1 -c 1 -o gpurun_out/${R}_gs $CMD > gpurun_out/${R}_ncu.log 2>&1
ls gpurun_out | grep $R
