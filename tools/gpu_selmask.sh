cd $GRAFT_REPO_ROOT
export SB200_LIB=$PWD/paper_1004_1741_b200/libsb200_exp.so
for rep in 1 2; do
for v in 0 1; do
  echo "SELMASK=$v rep=$rep" >> gpurun_out/selmask.log
  SB_SELMASK=$v python tools/probe.py --n 1024 --iters 40 --depths 4 --reps 3 >> gpurun_out/selmask.log 2>&1
  SB_SELMASK=$v python tools/probe.py --n 512 --iters 100 --depths 4 --reps 3 >> gpurun_out/selmask.log 2>&1
  SB_SELMASK=$v SB_SELF=1.05 python tools/probe.py --n 512 --iters 100 --depths 4 --reps 3 >> gpurun_out/selmask.log 2>&1
done
done
