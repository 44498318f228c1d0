cd $GRAFT_REPO_ROOT
export SB200_LIB=$PWD/paper_1004_1741_b200/libsb200_exp.so
for rep in 1 2; do
for v in 13 16 17; do
  echo "T3 JCFG=$v rep=$rep" >> gpurun_out/t3cfg.log
  SB_JCFG=$v timeout 120 python tools/probe.py --n 1024 --iters 48 --depths 3 --reps 3 >> gpurun_out/t3cfg.log 2>&1
  SB_JCFG=$v timeout 120 python tools/probe.py --n 512 --iters 99 --depths 3 --reps 3 >> gpurun_out/t3cfg.log 2>&1
done
for v in 20 22 23; do
  echo "T2 JCFG=$v rep=$rep" >> gpurun_out/t3cfg.log
  SB_JCFG=$v timeout 120 python tools/probe.py --n 1024 --iters 48 --depths 2 --reps 3 >> gpurun_out/t3cfg.log 2>&1
  SB_JCFG=$v timeout 120 python tools/probe.py --n 512 --iters 100 --depths 2 --reps 3 >> gpurun_out/t3cfg.log 2>&1
done
done
