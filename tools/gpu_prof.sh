cd $GRAFT_REPO_ROOT
R=${R:-r9}
python tools/probe.py --n 512 --iters 4 --depths 2,4 --reps 1 > gpurun_out/${R}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:jacobi_tb -s 2 -c 2 -o gpurun_out/${R}_jac python tools/probe.py --n 512 --iters 4 --depths 2,4 --reps 1 > gpurun_out/${R}_ncu_jac.log 2>&1
python tools/probe.py --n 256 --depths "" --gs --gs-iters 2 > gpurun_out/${R}_plain_gs.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gs_tile -s 2 -c 1 -o gpurun_out/${R}_gs python tools/probe.py --n 256 --depths "" --gs --gs-iters 2 > gpurun_out/${R}_ncu_gs.log 2>&1
python bench.py --steps 1 --warmup 3 --depth 2 --no-e2e --no-also --no-cpu > gpurun_out/${R}_bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 1 --warmup 3 --depth 2 --no-e2e --no-also --no-cpu > gpurun_out/${R}_ncu_launch.log 2>&1
ls -la gpurun_out/ | grep $R; tail -3 gpurun_out/${R}_ncu_jac.log gpurun_out/${R}_ncu_gs.log
