# A/B of two library builds: $A (default: the in-tree build) vs $B
cd $GRAFT_REPO_ROOT
A=${A:-$PWD/paper_1004_1741_b200/libsb200.so}; B=${B:-$PWD/paper_1004_1741_b200/libsb200_prev.so}
for rep in 1 2 3; do
  for L in $A $B; do
    echo "lib=$(basename $L) rep=$rep" >> gpurun_out/ab_lib.log
    SB200_LIB=$L timeout 120 python tools/probe.py --n 1024 --iters 40 --depths 4 --reps 3 >> gpurun_out/ab_lib.log 2>&1
    SB200_LIB=$L timeout 120 python tools/probe.py --n 512 --iters 100 --depths 3,4 --reps 3 >> gpurun_out/ab_lib.log 2>&1
  done
done
