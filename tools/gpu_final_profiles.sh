cd $GRAFT_REPO_ROOT
# Final-build evidence in one call: default bench (full line), the launch list
# of the plain bench command, and ncu --set full of the dominant kernels
# (Jacobi T=4 at 1024^3 from the bench command; T=1 and GS at 512^3 from the probe).
R=${R:-fin}
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?" >> gpurun_out/${R}_bench.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-also"
$CMD > gpurun_out/${R}_plain.json 2> gpurun_out/${R}_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 40 -c 1 -o gpurun_out/${R}_jacT4 $CMD > gpurun_out/${R}_ncu_jacT4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 2 -c 1 -o gpurun_out/${R}_jacT1 python tools/probe.py --n 512 --iters 8 --depths 1 > gpurun_out/${R}_ncu_jacT1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gs_tile -s 1 -c 1 -o gpurun_out/${R}_gs python tools/probe.py --n 512 --depths none --gs --gs-iters 20 > gpurun_out/${R}_ncu_gs.log 2>&1
for K in jacT4 jacT1 gs; do
  python tools/ncu_summary.py gpurun_out/${R}_${K}.ncu-rep > gpurun_out/${R}_${K}_summary.txt 2>&1
  ncu -i gpurun_out/${R}_${K}.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/${R}_${K}_raw.csv.gz
  [ $(stat -c %s gpurun_out/${R}_${K}.ncu-rep) -gt 15000000 ] && rm -f gpurun_out/${R}_${K}.ncu-rep
done
gzip -f gpurun_out/${R}_launches.csv
du -sh gpurun_out; tail -2 gpurun_out/${R}_bench.err
