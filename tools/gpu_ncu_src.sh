cd $GRAFT_REPO_ROOT
# full ncu capture (with source) of one temporally blocked Jacobi launch
R=${R:-src}
N=${N:-1024}; D=${D:-4}
python tools/probe.py --n $N --iters $D --depths $D --reps 1 > gpurun_out/${R}_plain.log 2>&1 || { tail gpurun_out/${R}_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 1 -c 1 -o gpurun_out/${R} python tools/probe.py --n $N --iters $D --depths $D --reps 2 > gpurun_out/${R}_ncu.log 2>&1
tail -3 gpurun_out/${R}_ncu.log
ls -la gpurun_out/${R}*
