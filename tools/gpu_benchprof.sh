cd $GRAFT_REPO_ROOT
R=${R:-r40}
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-also"
$CMD > gpurun_out/${R}_plain.json 2> gpurun_out/${R}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 40 -c 1 -o gpurun_out/${R}_jac $CMD > gpurun_out/${R}_ncu_full.log 2>&1
ls -la gpurun_out | grep $R; tail -3 gpurun_out/${R}_ncu_full.log
# summaries on the box; keep the report only if it fits the copy-back limit
python tools/ncu_summary.py gpurun_out/${R}_jac.ncu-rep > gpurun_out/${R}_jac_summary.txt 2>&1
ncu -i gpurun_out/${R}_jac.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${R}_jac_raw.csv.gz
[ $(stat -c %s gpurun_out/${R}_jac.ncu-rep) -gt 30000000 ] && rm -f gpurun_out/${R}_jac.ncu-rep
gzip -f gpurun_out/${R}_launches.csv
du -sh gpurun_out
