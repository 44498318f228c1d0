cd $GRAFT_REPO_ROOT
# full ncu capture (with source) of one Gauss-Seidel launch (512^3, $IT sweeps)
R=${R:-gs}
IT=${IT:-20}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-gs_tile} -s 1 -c 1 -o gpurun_out/${R} python tools/probe.py --n 512 --depths none --gs --gs-iters $IT > gpurun_out/${R}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${R}.ncu-rep > gpurun_out/${R}_summary.txt 2>&1
ncu -i gpurun_out/${R}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${R}_src.csv.gz
[ $(stat -c %s gpurun_out/${R}.ncu-rep) -gt 30000000 ] && rm -f gpurun_out/${R}.ncu-rep
du -sh gpurun_out
