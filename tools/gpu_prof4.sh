cd $GRAFT_REPO_ROOT
R=${R:-r42}
for cfg in ${CFGS:-"0 3" "1 4"}; do set -- ${cfg/_/ }
CMD="python tools/probe.py --n ${N:-1024} --iters $2 --depths $2 --reps 1"
SB_JCFG=$1 timeout 300 $CMD > gpurun_out/${R}_plain_$1_$2.log 2>&1 && \
SB_JCFG=$1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 1 -c 1 -o gpurun_out/${R}_jac_v$1_T$2 $CMD > gpurun_out/${R}_ncu_$1_$2.log 2>&1
done
ls gpurun_out | grep $R
